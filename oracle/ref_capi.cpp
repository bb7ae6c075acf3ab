// TEST INFRASTRUCTURE ONLY — C entry points over the REFERENCE's own oracle,
// compiled unmodified from /root/reference/proj/src/{fpbits,oracle}.cpp by
// the `ref` target of oracle/Makefile into oracle/_ref/libcrvec_ref.so. Used to pin the C
// restatement (oracle/crvec_oracle.c) and as the reference CPU arm of bench.py.
// ref: proj/include/crvec/oracle.hpp:74-90, proj/include/crvec/fpbits.hpp:131.
#include <atomic>
#include <cstdint>
#include <cstring>
#include <thread>
#include <vector>

#include "crvec/fpbits.hpp"
#include "crvec/oracle.hpp"

using namespace crvec;

extern "C" {

uint32_t crvec_ref_ziv_f32(int f, uint32_t x, int mode, int start_prec, int* prec) {
  try {
    auto r = ziv_correctly_round_f32(static_cast<FuncId>(f), Binary32(x),
                                     static_cast<RoundingMode>(mode), start_prec);
    if (prec) *prec = r.decided_at_precision;
    return r.value.bits;
  } catch (...) {
    if (prec) *prec = -1;
    return 0x7FC00000u;
  }
}

uint64_t crvec_ref_ziv_f64(int f, uint64_t x, int mode, int start_prec, int* prec) {
  try {
    auto r = ziv_correctly_round_f64(static_cast<FuncId>(f), Binary64(x),
                                     static_cast<RoundingMode>(mode), start_prec);
    if (prec) *prec = r.decided_at_precision;
    return r.value.bits;
  } catch (...) {
    if (prec) *prec = -1;
    return 0x7FF8000000000000ull;
  }
}

int crvec_ref_all_modes_f32(int f, uint32_t x, uint32_t* out) {
  try {
    auto r = oracle_all_modes_f32(static_cast<FuncId>(f), Binary32(x));
    for (int m = 0; m < 4; ++m) out[m] = r.value[m].bits;
    return 0;
  } catch (...) {
    return -1;
  }
}

int crvec_ref_all_modes_f64(int f, uint64_t x, uint64_t* out) {
  try {
    auto r = oracle_all_modes_f64(static_cast<FuncId>(f), Binary64(x));
    for (int m = 0; m < 4; ++m) out[m] = r.value[m].bits;
    return 0;
  } catch (...) {
    return -1;
  }
}

uint32_t crvec_ref_convert_f64_to_f32(uint64_t v, int mode) {
  return convert_f64_to_f32(Binary64(v), static_cast<RoundingMode>(mode)).bits;
}

// Reference CPU path over an array: ziv_correctly_round_f32 per element (the
// reference's only correct binary32 path), std::thread over 2^20-element
// chunks (ref: SPEC.md chunking rule). Returns 0, or -1 if any element hit the
// precision cap.
int crvec_ref_batch_f32(int f, const uint32_t* x, uint32_t* y, uint64_t n, int mode,
                        int threads) {
  if (threads <= 0) threads = static_cast<int>(std::thread::hardware_concurrency());
  if (threads <= 0) threads = 1;
  std::atomic<uint64_t> next{0};
  std::atomic<int> rc{0};
  const uint64_t grain = 4096;
  auto work = [&]() {
    for (;;) {
      uint64_t b = next.fetch_add(grain);
      if (b >= n) break;
      uint64_t e = b + grain < n ? b + grain : n;
      for (uint64_t i = b; i < e; ++i) {
        try {
          y[i] = ziv_correctly_round_f32(static_cast<FuncId>(f), Binary32(x[i]),
                                         static_cast<RoundingMode>(mode))
                     .value.bits;
        } catch (...) {
          rc = -1;
        }
      }
    }
  };
  std::vector<std::thread> ts;
  for (int t = 1; t < threads; ++t) ts.emplace_back(work);
  work();
  for (auto& t : ts) t.join();
  return rc.load();
}

int crvec_ref_batch_f64(int f, const uint64_t* x, uint64_t* y, uint64_t n, int mode,
                        int threads) {
  if (threads <= 0) threads = static_cast<int>(std::thread::hardware_concurrency());
  if (threads <= 0) threads = 1;
  std::atomic<uint64_t> next{0};
  std::atomic<int> rc{0};
  auto work = [&]() {
    for (;;) {
      uint64_t b = next.fetch_add(256);
      if (b >= n) break;
      uint64_t e = b + 256 < n ? b + 256 : n;
      for (uint64_t i = b; i < e; ++i) {
        try {
          y[i] = ziv_correctly_round_f64(static_cast<FuncId>(f), Binary64(x[i]),
                                         static_cast<RoundingMode>(mode))
                     .value.bits;
        } catch (...) {
          rc = -1;
        }
      }
    }
  };
  std::vector<std::thread> ts;
  for (int t = 1; t < threads; ++t) ts.emplace_back(work);
  work();
  for (auto& t : ts) t.join();
  return rc.load();
}

int crvec_ref_boundary_distance_f32(int f, uint32_t x, double *dist, int *exact, int *domain) {
  auto d = boundary_distance_f32(static_cast<FuncId>(f), Binary32(x));
  *dist = d.scaled_distance;
  *exact = d.exact;
  *domain = d.domain;
  return 0;
}

int crvec_ref_boundary_distance_f64(int f, uint64_t x, double *dist, int *exact, int *domain) {
  auto d = boundary_distance_f64(static_cast<FuncId>(f), Binary64(x));
  *dist = d.scaled_distance;
  *exact = d.exact;
  *domain = d.domain;
  return 0;
}

uint64_t crvec_ref_hardest_case_search(int f, uint32_t lo, uint32_t hi, uint32_t *out_bits,
                                       double *out_dist, uint64_t cap) {
  auto v = hardest_case_search(static_cast<FuncId>(f), lo, hi, 0);
  uint64_t m = (cap && cap < v.size()) ? cap : v.size();
  if (out_bits)
    for (uint64_t i = 0; i < m; ++i) {
      out_bits[i] = v[i].input_bits;
      out_dist[i] = v[i].scaled_distance;
    }
  return v.size();
}

// Exhaustive-sweep golden hashes straight from the reference's oracle:
// for chunks [chunk_lo, chunk_hi) of 2^20 binary32 patterns,
//   h[(c - chunk_lo)*4 + m] = sum_p mix64((oracle_all_modes_f32(f, p)[m] << 32) | p)
// (the hash of include/crvec.h crvec_sweep_f32 / oracle/crvec_oracle.c).
// oracle_all_modes_f32 is ref: proj/src/oracle.cpp:347-388, unmodified.
// Returns the number of patterns whose oracle call threw (precision cap).
static inline uint64_t ref_mix64(uint64_t z) {
  z ^= z >> 30;
  z *= 0xbf58476d1ce4e5b9ull;
  z ^= z >> 27;
  z *= 0x94d049bb133111ebull;
  z ^= z >> 31;
  return z;
}

uint64_t crvec_ref_sweep_hashes(int f, uint32_t chunk_lo, uint32_t chunk_hi, uint64_t* h,
                                int threads) {
  if (threads <= 0) threads = static_cast<int>(std::thread::hardware_concurrency());
  if (threads <= 0) threads = 1;
  const uint32_t nchunks = chunk_hi - chunk_lo;
  std::atomic<uint32_t> next{0};
  std::atomic<uint64_t> fails{0};
  auto work = [&]() {
    for (;;) {
      const uint32_t i = next.fetch_add(1);
      if (i >= nchunks) break;
      const uint32_t c = chunk_lo + i;
      uint64_t acc[4] = {0, 0, 0, 0};
      for (uint32_t k = 0; k < (1u << 20); ++k) {
        const uint32_t p = (c << 20) | k;
        uint32_t o[4] = {0x7FC00000u, 0x7FC00000u, 0x7FC00000u, 0x7FC00000u};
        try {
          auto r = oracle_all_modes_f32(static_cast<FuncId>(f), Binary32(p));
          for (int m = 0; m < 4; ++m) o[m] = r.value[m].bits;
        } catch (...) {
          fails.fetch_add(1);
        }
        for (int m = 0; m < 4; ++m) acc[m] += ref_mix64((static_cast<uint64_t>(o[m]) << 32) | p);
      }
      std::memcpy(h + 4ull * i, acc, sizeof(acc));
    }
  };
  std::vector<std::thread> ts;
  for (int t = 1; t < threads; ++t) ts.emplace_back(work);
  work();
  for (auto& t : ts) t.join();
  return fails.load();
}

}  // extern "C"
