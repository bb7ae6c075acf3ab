// Kernel templates: streaming map kernels (128/256-bit coalesced I/O, block-
// uniform grid-stride loops so register tables can use __shfl_sync), the
// warp-uniform Payne-Hanek reduction, the rare accurate-path fallback, and the
// exhaustive-sweep kernel with a commutative per-chunk hash.
#pragma once
#include <cuda_runtime.h>

#include <cstdlib>

#include "crvec_fns_f32.cuh"

namespace crvec {

constexpr int kThreads = 256;
constexpr int kWarps = kThreads / 32;
constexpr unsigned kFull = 0xffffffffu;

template <class F>
struct IsTrig {
  static constexpr bool value = false;
};
template <int W>
struct IsTrig<FnTrig<W>> {
  static constexpr bool value = true;
};

// Streaming 128-bit accesses: read-only non-coherent path without L1
// allocation, evict-first stores (inputs and outputs are touched once).
__device__ __forceinline__ float4 ld_stream(const float4 *p) {
  float4 v;
  asm volatile("ld.global.nc.L1::no_allocate.v4.f32 {%0,%1,%2,%3}, [%4];"
               : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
               : "l"(p));
  return v;
}
__device__ __forceinline__ void st_stream(float4 *p, float4 v) {
  asm volatile("st.global.cs.v4.f32 [%0], {%1,%2,%3,%4};" ::"l"(p), "f"(v.x), "f"(v.y), "f"(v.z),
               "f"(v.w)
               : "memory");
}

// Per-lane access unit of the map kernels: VW consecutive floats, one 128-bit
// (VW = 4) or 256-bit (VW = 8: LDG/STG.E.ENL2.256, new on sm_100) access, so a
// warp moves 512 B or 1 KiB per instruction.
template <int VW>
struct alignas(4 * VW) Vec {
  float v[VW];
};
template <int VW>
__device__ __forceinline__ Vec<VW> ld_vec(const Vec<VW> *p) {
  Vec<VW> r;
  if constexpr (VW == 4) {
    asm volatile("ld.global.nc.L1::no_allocate.v4.f32 {%0,%1,%2,%3}, [%4];"
                 : "=f"(r.v[0]), "=f"(r.v[1]), "=f"(r.v[2]), "=f"(r.v[3])
                 : "l"(p));
  } else {
    static_assert(VW == 8, "VW");
    asm volatile("ld.global.nc.L1::no_allocate.v8.f32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=f"(r.v[0]), "=f"(r.v[1]), "=f"(r.v[2]), "=f"(r.v[3]), "=f"(r.v[4]),
                   "=f"(r.v[5]), "=f"(r.v[6]), "=f"(r.v[7])
                 : "l"(p));
  }
  return r;
}
template <int VW>
__device__ __forceinline__ void st_vec(Vec<VW> *p, const uint32_t *y) {
  if constexpr (VW == 4) {
    asm volatile("st.global.cs.v4.b32 [%0], {%1,%2,%3,%4};" ::"l"(p), "r"(y[0]), "r"(y[1]),
                 "r"(y[2]), "r"(y[3])
                 : "memory");
  } else {
    asm volatile("st.global.cs.v8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"l"(p), "r"(y[0]),
                 "r"(y[1]), "r"(y[2]), "r"(y[3]), "r"(y[4]), "r"(y[5]), "r"(y[6]), "r"(y[7])
                 : "memory");
  }
}

// Accurate path: one lane, double-double evaluation + round_dd. Out of line so
// the fast path keeps its register budget; reached with probability ~2^-24.
template <class F, int M>
__device__ __noinline__ uint32_t slow_round(float x) {
  DD v = F::slow(x);
  return round_dd<M>(v.hi, v.lo);
}
template <class F>
__device__ __noinline__ DD slow_dd(float x) {
  return F::slow(x);
}

// ------------------------------------------------ trig argument reduction
// Warp-uniform Payne-Hanek: while no lane of the warp's step holds a large
// argument (|x| >= 2^12) every lane takes the two-part Cody-Waite reduction;
// as soon as one does, the whole warp takes the exponent-indexed Payne-Hanek
// reduction (red_trig_ph: the bits of 16/pi that matter for x's exponent,
// one 16-byte shared-table row, 4 FP64 operations + the pi/16 scaling),
// which is exact for small arguments too. No compaction, no queue, no
// divergence: round 1's per-warp ballot queue cost ~25 thread-instructions
// per element on the config-3 mix (profiles/r02/ncu_lines_sinf.txt).
struct PHBlock {
  double tab[512];  // PH_T by biased exponent b: hi at [b], lo at [256 + b]
};

template <int NE>
__device__ __forceinline__ void trig_reduce(const float (&xs)[NE], RedTrig (&q)[NE], const PHBlock *sh) {
#ifndef CRVEC_TRIG_UNIFIED
  float mx = 0.0f;  // NaN lanes are ignored by fmaxf (they are rare lanes either way)
#pragma unroll
  for (int e = 0; e < NE; ++e) mx = fmaxf(mx, fabsf(xs[e]));
  if (!__any_sync(kFull, mx >= 0x1p12f)) {
#pragma unroll
    for (int e = 0; e < NE; ++e) q[e] = red_trig_small(f2d(xs[e]));
    return;
  }
#endif
#pragma unroll
  for (int e = 0; e < NE; ++e) q[e] = red_trig_ph(xs[e], sh->tab);
}

// Fast results for NE elements per lane (warp converged on entry).
template <class F, int NE>
__device__ __forceinline__ void fast_lanes(const float (&xs)[NE], Fast (&f)[NE],
                                           const typename F::Regs &R, PHBlock *sh) {
  if constexpr (IsTrig<F>::value) {
    RedTrig q[NE];
    trig_reduce<NE>(xs, q, sh);
#pragma unroll
    for (int e = 0; e < NE; ++e) f[e] = F::from_red(xs[e], q[e], R);
  } else {
#pragma unroll
    for (int e = 0; e < NE; ++e) f[e] = F::fast(xs[e], R);
  }
}


// Rare bit of one slot, OR-ed into `mask` with one predicated OR: the lane is
// undecided by the rounding test (near_boundary on the low word of `a`) or x
// is outside the function's main range kLo < v <= kHi, v = |x| (kMainAbs) or
// x, tested with unordered float compares so NaN is rare; functions with a
// tiny rule also drop tiny lanes (|x| <= kTiny, the rule is applied to the
// result bits). One predicate chain: VIADD, LOP3.P, 2-3 FSETP, predicated
// VIADD (the bool form, (!main | nb) << e, compiles to 2-5 SEL per element).
// The float range is the same set as F::in_main (integer form, used by the
// rare path and the sweep kernels); the exhaustive map-kernel sweep checks it.
template <class F, class = void>
struct HasTiny { static constexpr bool value = false; };
template <class F>
struct HasTiny<F, decltype((void)F::kTiny)> { static constexpr bool value = true; };

template <class F, class = void>
struct HasMainRange { static constexpr bool value = false; };
template <class F>
struct HasMainRange<F, decltype((void)F::kMainAbs)> { static constexpr bool value = true; };

template <class F>
__device__ __forceinline__ void rare_or(unsigned &mask, double a, float x, unsigned bit) {
  constexpr uint32_t W = 0x0FFFFFFFu & ~(4u * F::E - 1u);
  const float v = F::kMainAbs ? fabsf(x) : x;
  if constexpr (HasTiny<F>::value) {
    asm("{\n\t.reg .pred p;\n\t.reg .u32 t;\n\t"
        "add.u32 t, %1, %4;\n\t"
        "and.b32 t, t, %5;\n\t"
        "setp.eq.u32 p, t, 0;\n\t"
        "setp.leu.or.f32 p, %2, %6, p;\n\t"
        "setp.gtu.or.f32 p, %2, %7, p;\n\t"
        "setp.gtu.and.f32 p, %8, %9, p;\n\t"
        "@p or.b32 %0, %0, %3;\n\t}"
        : "+r"(mask)
        : "r"(d2lo(a)), "f"(v), "r"(bit), "n"(2u * F::E), "n"(W), "f"(F::kMainLo), "f"(F::kMainHi),
          "f"(fabsf(x)), "f"(F::kTiny));
  } else {
    asm("{\n\t.reg .pred p;\n\t.reg .u32 t;\n\t"
        "add.u32 t, %1, %4;\n\t"
        "and.b32 t, t, %5;\n\t"
        "setp.eq.u32 p, t, 0;\n\t"
        "setp.leu.or.f32 p, %2, %6, p;\n\t"
        "setp.gtu.or.f32 p, %2, %7, p;\n\t"
        "@p or.b32 %0, %0, %3;\n\t}"
        : "+r"(mask)
        : "r"(d2lo(a)), "f"(v), "r"(bit), "n"(2u * F::E), "n"(W), "f"(F::kMainLo), "f"(F::kMainHi));
  }
}

// Common path for NE elements per lane: fast approximation, one static-mode
// conversion, and the per-lane mask of rare slots (bit e: slot e is outside
// the main range, or undecided by the rounding test).
template <class F, int M, int NE>
__device__ __forceinline__ unsigned fast_eval(const float (&xs)[NE], uint32_t (&ys)[NE],
                                              const typename F::Regs &R, PHBlock *sh) {
  static_assert((F::E & (F::E - 1)) == 0 && F::E <= (1u << 24), "E: power of two");
  Fast f[NE];
  fast_lanes<F, NE>(xs, f, R, sh);
  unsigned mask = 0;
#pragma unroll
  for (int e = 0; e < NE; ++e) {
    ys[e] = f2u(cvt_f32<M>(f[e].a));
    if constexpr (HasMainRange<F>::value) {
      rare_or<F>(mask, f[e].a, xs[e], 1u << e);
    } else {  // bool form (expm1f: the predicate chain measured 2% slower there)
      const bool rare = (!f[e].main) | near_boundary(f[e].a, F::E);
      mask |= (unsigned)rare << e;
    }
    if constexpr (HasTiny<F>::value)  // log1pf: tiny-argument rule on the result bits
      ys[e] = fabsf(xs[e]) <= F::kTiny ? F::template tiny_bits<M>(f2u(xs[e])) : ys[e];
  }
  return mask;
}

// One rare lane value: IEEE special / tiny / saturation rule, or the
// double-double accurate path (counted).
template <class F, int M>
__device__ __forceinline__ uint32_t resolve_one(float x, int &cnt) {
  if (F::in_main(f2u(x))) {
    ++cnt;
    return slow_round<F, M>(x);
  }
  return F::template special<M>(x);
}

template <int NE>
__device__ __forceinline__ float gather_slot(const float (&xs)[NE], unsigned low) {
  float xe = xs[0];
#pragma unroll
  for (int e = 1; e < NE; ++e) xe = (low >> e) & 1u ? xs[e] : xe;
  return xe;
}

// Rare path (register form, scalar kernels): each pass takes every lane's
// lowest pending slot, gathers its input with selects (no dynamic register
// indexing), resolves it and scatters the result back; a lane rarely has two
// pending slots, so one pass usually serves the whole warp.
template <class F, int M, int NE>
__device__ __forceinline__ void resolve_rare(const float (&xs)[NE], uint32_t (&ys)[NE], unsigned mask,
                                             unsigned long long *counters) {
  int cnt = 0;
  do {
    const unsigned low = mask & (0u - mask);
    const float xe = gather_slot<NE>(xs, low);
    uint32_t r = 0;
    if (low) r = resolve_one<F, M>(xe, cnt);
#pragma unroll
    for (int e = 0; e < NE; ++e) ys[e] = (low >> e) & 1u ? r : ys[e];
    mask &= ~low;
  } while (__any_sync(kFull, mask != 0));
  if (cnt) atomicAdd(counters, (unsigned long long)cnt);
}

// Rare path (store form, map kernels): runs after the vector stores; each
// pass gathers every lane's lowest pending input from registers, resolves it
// and overwrites the one output float with a scalar store (same thread,
// program order), so no scatter back into the register results is needed.
// In-place calls are safe: the inputs are still in registers.
// fbase (the lane's first float index) is 64-bit: a launch covers up to
// kMaxNV vectors of VW floats, more than 2^32 floats.
template <class F, int M, int NE, int VW>
__device__ __forceinline__ void resolve_rare_store(const float (&xs)[NE], unsigned mask, float *yf,
                                                   uint64_t fbase, unsigned long long *counters) {
  int cnt = 0;
  do {
    const unsigned low = mask & (0u - mask);
    const float xe = gather_slot<NE>(xs, low);
    if (low) {
      static_assert((NE & (NE - 1)) == 0, "NE: power of two");
      // unsigned and bounded (mask has NE bits): / and % fold to shifts and masks
      const uint32_t e = ((uint32_t)__ffs(mask) - 1u) & (NE - 1u);
      yf[fbase + (32u * VW * (e / VW) + (e % VW))] = u2f(resolve_one<F, M>(xe, cnt));
    }
    mask &= ~low;
  } while (__any_sync(kFull, mask != 0));
  if (cnt) atomicAdd(counters, (unsigned long long)cnt);
}

// Rare path (staged form): the warp's lanes with pending slots write their NE
// inputs to a per-thread shared-memory row (NE/4 128-bit stores) and each
// resolves its own pending slots in a divergent loop (no select gather, no
// warp-wide pass per slot depth), overwriting the one output float.
template <class F, int M, int NE, int VW>
__device__ __forceinline__ void resolve_rare_staged(const float (&xs)[NE], unsigned mask, float *yf,
                                                    uint64_t fbase, unsigned long long *counters) {
  __shared__ float4 stage[kThreads * (NE / 4)];
  if (mask) {
    float4 *row = stage + threadIdx.x * (NE / 4);
#pragma unroll
    for (int k = 0; k < NE / 4; ++k) row[k] = make_float4(xs[4 * k], xs[4 * k + 1], xs[4 * k + 2], xs[4 * k + 3]);
    const float *rf = reinterpret_cast<const float *>(row);
    float *yl = yf + fbase;  // the lane's first output float: one 64-bit add per step
    asm("" : "+l"(yl));      // keep it: slot offsets are then 32-bit (one IMAD.WIDE per store)
    int cnt = 0;
    do {
      // highest pending slot first: one FLO (no bit reverse), 32-bit offsets
      const uint32_t e = 31u - (uint32_t)__clz((int)mask);
      const uint32_t v = resolve_one<F, M>(rf[e], cnt);
      asm volatile("st.global.b32 [%0], %1;" ::"l"(yl + (32u * VW * (e / VW) + (e % VW))), "r"(v) : "memory");
      mask ^= 1u << e;
    } while (mask);
    if (cnt) atomicAdd(counters, (unsigned long long)cnt);
  }
}
template <class F> struct RareStaged { static constexpr bool value = false; };
template <int B> struct RareStaged<FnLogB<B>> { static constexpr bool value = true; };
template <> struct RareStaged<FnLog1p> { static constexpr bool value = true; };
template <> struct RareStaged<FnTanh> { static constexpr bool value = true; };
template <> struct RareStaged<FnSinh> { static constexpr bool value = true; };

template <class F, int M, int NE>
__device__ __forceinline__ void eval_lanes(const float (&xs)[NE], uint32_t (&ys)[NE],
                                           const typename F::Regs &R, PHBlock *sh,
                                           unsigned long long *counters) {
  const unsigned mask = fast_eval<F, M, NE>(xs, ys, R, sh);
  if (__any_sync(kFull, mask != 0)) resolve_rare<F, M, NE>(xs, ys, mask, counters);
}

// The Payne-Hanek table exists only in the trig kernels (4 KB per block).
template <class F>
__device__ __forceinline__ PHBlock *ph_storage() {
  if constexpr (IsTrig<F>::value) {
    __shared__ PHBlock sh;
    for (int i = threadIdx.x; i < 256; i += blockDim.x) {
      sh.tab[i] = PH_T[2 * i];
      sh.tab[256 + i] = PH_T[2 * i + 1];
    }
    __syncthreads();
    return &sh;
  } else {
    return nullptr;
  }
}

// ------------------------------------------------------------ map kernels ----
// NV vectors of VW floats per lane per step; the loop trip count is warp-
// uniform so the register-table shuffles always see a full warp.
// Kernel shape per function, chosen by measurement (tools/gpu_ab2.sh over
// tools/mk_shape_variants.sh / mk_tune_variants.sh builds;
// profiles/r01/shapes_sw2.txt, tune_*.txt): vector width (vw 4: 128-bit,
// vw 8: 256-bit accesses), vectors per lane per step (nv) and the
// __launch_bounds__ min-blocks register cap (minb; 256 threads per block).
// Rare-path form per function (measured, profiles/r01/ab_rare_store.txt,
// profiles/r01/tune_store_form.txt, profiles/r01/tune_vw8.txt):
// store form (resolve after the vector store, scalar overwrite) or register
// form (gather + scatter before the store); within the store form, the staged
// variant (RareStaged above: shared-memory row + per-lane loop, round 2,
// profiles/r02/ab_log_rare.txt, ab_other.txt) for the log family, tanh, sinh.
// The choice changes the main path's register allocation, so it is taken per
// kernel; shapes re-measured in round 2 (log1pf, expm1f 8:2:2).
template <class F> struct RareStore { static constexpr bool value = false; };
template <int B> struct RareStore<FnLogB<B>> { static constexpr bool value = true; };
template <bool A> struct RareStore<FnAsinAcos<A>> { static constexpr bool value = true; };
template <> struct RareStore<FnExpm1> { static constexpr bool value = true; };
template <> struct RareStore<FnRsqrt> { static constexpr bool value = true; };
template <> struct RareStore<FnTanh> { static constexpr bool value = true; };
template <> struct RareStore<FnLog1p> { static constexpr bool value = true; };
template <> struct RareStore<FnSinh> { static constexpr bool value = true; };
template <int W> struct RareStore<FnTrig<W>> { static constexpr bool value = true; };

// L2 bulk prefetch (cp.async.bulk.prefetch.L2, one lane per warp) of the
// warp's inputs two grid-stride steps ahead: the register double buffer keeps
// one step (2 KiB per warp) in flight, ~32 KiB per SM at these occupancies,
// which is short of what HBM latency x bandwidth needs; the L2 copy turns the
// next-step loads into L2 hits. Measured per function (profiles/r02/
// ab_prefetch.txt): exp/exp2/exp10/expm1, the log family and cosh
// +1.5..3.5% per launch; issue-bound kernels (trig, inverse trig, sinh, tanh)
// and rsqrt lose 1-4%, so they go without it.
template <class F> struct PrefetchL2 { static constexpr bool value = false; };
template <> struct PrefetchL2<FnExp> { static constexpr bool value = true; };
template <> struct PrefetchL2<FnExp2> { static constexpr bool value = true; };
template <> struct PrefetchL2<FnExp10> { static constexpr bool value = true; };
template <> struct PrefetchL2<FnExpm1> { static constexpr bool value = true; };
template <int B> struct PrefetchL2<FnLogB<B>> { static constexpr bool value = true; };
template <> struct PrefetchL2<FnLog1p> { static constexpr bool value = true; };
template <> struct PrefetchL2<FnCosh> { static constexpr bool value = true; };
// end of round 2: sinh +4.7%, atan / asin / acos +0.5..1% (tanh and trig lose
// 1-3%; profiles/r02/ab_prefetch_r3b.txt)
template <> struct PrefetchL2<FnSinh> { static constexpr bool value = true; };
template <> struct PrefetchL2<FnAtan> { static constexpr bool value = true; };
template <bool A> struct PrefetchL2<FnAsinAcos<A>> { static constexpr bool value = true; };

template <class F>
struct KernelShape {
  static constexpr int vw = 4, nv = 2, minb = 3;
};
template <> struct KernelShape<FnExp2> { static constexpr int vw = 8, nv = 1, minb = 3; };
template <> struct KernelShape<FnExp10> { static constexpr int vw = 8, nv = 1, minb = 3; };
template <> struct KernelShape<FnExp> { static constexpr int vw = 8, nv = 1, minb = 3; };
template <> struct KernelShape<FnExpm1> { static constexpr int vw = 8, nv = 2, minb = 2; };
// tanh, asin/acos: 8:2:2 after the 4-op division / 5-op sqrt (+1.2..2.7%,
// profiles/r02/ab_shapes_r2w.txt; the trig kernels lose 3-7% at 8:2:2)
template <> struct KernelShape<FnTanh> { static constexpr int vw = 8, nv = 2, minb = 2; };
template <> struct KernelShape<FnLog1p> { static constexpr int vw = 8, nv = 2, minb = 2; };
template <> struct KernelShape<FnLog> { static constexpr int vw = 8, nv = 2, minb = 2; };
template <> struct KernelShape<FnLog2> { static constexpr int vw = 8, nv = 2, minb = 2; };
template <> struct KernelShape<FnSinh> { static constexpr int vw = 8, nv = 2, minb = 2; };
template <> struct KernelShape<FnCosh> { static constexpr int vw = 8, nv = 2, minb = 2; };
template <> struct KernelShape<FnLog10> { static constexpr int vw = 8, nv = 2, minb = 2; };
template <> struct KernelShape<FnAtan> { static constexpr int vw = 8, nv = 2, minb = 2; };
template <> struct KernelShape<FnRsqrt> { static constexpr int vw = 8, nv = 1, minb = 4; };
template <bool A> struct KernelShape<FnAsinAcos<A>> { static constexpr int vw = 8, nv = 2, minb = 2; };
template <int W> struct KernelShape<FnTrig<W>> { static constexpr int vw = 8, nv = 1, minb = 3; };

// One grid-stride step of the map kernel: issue the loads of the next step
// into `nxt`, evaluate `cur`, store. Called alternately with the two register
// buffers swapped, so the double buffer needs no register moves.
template <class F, int M, int VW, int NV>
__device__ __forceinline__ void map_step(const Vec<VW> *__restrict__ x, Vec<VW> *__restrict__ y,
                                         uint32_t nv, uint32_t base, uint32_t ub, uint32_t stride,
                                         const Vec<VW> (&cur)[NV], Vec<VW> (&nxt)[NV],
                                         const typename F::Regs &R, PHBlock *sh,
                                         unsigned long long *counters) {
  float xs[VW * NV];
  if constexpr (PrefetchL2<F>::value) {
    // the block's inputs two steps ahead into L2: one bulk prefetch by thread 0,
    // from the block base ub (uniform: blockIdx, stride), so the operands sit
    // in uniform registers (a per-warp address derived from threadIdx made
    // ptxas wrap the instruction in a waterfall loop, ~10 instructions)
    const uint32_t pb = ub + 2u * stride;
    if (threadIdx.x == 0 && pb + (uint32_t)(kThreads * NV) <= nv)
      asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(x + pb),
                   "r"((uint32_t)(kThreads * NV * sizeof(Vec<VW>)))
                   : "memory");
  }
#pragma unroll
  for (int k = 0; k < NV; ++k) {
    const uint32_t in = base + stride + 32 * k;
    if (in < nv) nxt[k] = ld_vec<VW>(x + in);
#pragma unroll
    for (int j = 0; j < VW; ++j) xs[VW * k + j] = cur[k].v[j];
  }
  uint32_t ys[VW * NV];
  if constexpr (RareStore<F>::value) {
    unsigned mask = fast_eval<F, M, VW * NV>(xs, ys, R, sh);
#pragma unroll
    for (int k = 0; k < NV; ++k) {
      const uint32_t i = base + 32 * k;
      if (i < nv) st_vec<VW>(y + i, ys + VW * k);
      else mask &= ~(((1u << VW) - 1u) << (VW * k));  // stale inputs past the end
    }
    if (__any_sync(kFull, mask != 0)) {
      if constexpr (RareStaged<F>::value)
        resolve_rare_staged<F, M, VW * NV, VW>(xs, mask, (float *)y, (uint64_t)VW * base, counters);
      else
        resolve_rare_store<F, M, VW * NV, VW>(xs, mask, (float *)y, (uint64_t)VW * base, counters);
    }
  } else {
    unsigned mask = fast_eval<F, M, VW * NV>(xs, ys, R, sh);
#pragma unroll
    for (int k = 0; k < NV; ++k)  // stale inputs past the end
      if (base + 32 * k >= nv) mask &= ~(((1u << VW) - 1u) << (VW * k));
    if (__any_sync(kFull, mask != 0)) resolve_rare<F, M, VW * NV>(xs, ys, mask, counters);
#pragma unroll
    for (int k = 0; k < NV; ++k) {
      const uint32_t i = base + 32 * k;
      if (i < nv) st_vec<VW>(y + i, ys + VW * k);
    }
  }
}

template <class F, int M>
__global__ void __launch_bounds__(kThreads, KernelShape<F>::minb)
    k_map_vec(const float *__restrict__ xf, float *__restrict__ yf, uint32_t nv,
              unsigned long long *counters) {
  constexpr int VW = KernelShape<F>::vw, NV = KernelShape<F>::nv;
  const Vec<VW> *x = reinterpret_cast<const Vec<VW> *>(xf);
  Vec<VW> *y = reinterpret_cast<Vec<VW> *>(yf);
  PHBlock *sh = ph_storage<F>();
  typename F::Regs R;
  F::load(R);
  // 32-bit vector indices (the launcher keeps nv <= 2^31): one IMAD.WIDE per
  // address, one compare per access. Each warp handles NV x 32 vectors per
  // step; the trip count is warp-uniform (register-table shuffles need the
  // whole warp).
  const uint32_t lane = threadIdx.x & 31;
  const uint32_t stride = gridDim.x * (uint32_t)(kThreads * NV);
  uint32_t base = ((blockIdx.x * kThreads + threadIdx.x) >> 5) * (32 * NV) + lane;
  Vec<VW> va[NV], vb[NV];
#pragma unroll
  for (int k = 0; k < NV; ++k) {
#pragma unroll
    for (int j = 0; j < VW; ++j) va[k].v[j] = 1.0f;
    vb[k] = va[k];
    if (base + 32 * k < nv) va[k] = ld_vec<VW>(x + base + 32 * k);
  }
  // block-uniform loop over ub, the block's first vector of the step (kept in
  // uniform registers: the L2 prefetch's operands need no waterfall loop); a
  // warp whose part of the last step lies past nv skips it (warp-uniform test)
  // block-uniform loop over ub, the block's first vector of the step (kept in
  // uniform registers: the L2 prefetch's operands need no waterfall loop); a
  // warp whose part of the last step lies past nv runs it with every load,
  // store and rare slot masked off
  const uint32_t wofs = base - blockIdx.x * (uint32_t)(kThreads * NV);  // warp offset + lane
  for (uint32_t ub = blockIdx.x * (uint32_t)(kThreads * NV); ub < nv; ub += 2u * stride) {
    map_step<F, M, VW, NV>(x, y, nv, ub + wofs, ub, stride, va, vb, R, sh, counters);
    if (ub + stride >= nv) break;
    map_step<F, M, VW, NV>(x, y, nv, ub + stride + wofs, ub + stride, stride, vb, va, R, sh, counters);
  }
}

// Any alignment / tails: one element per lane.
template <class F, int M>
__global__ void __launch_bounds__(kThreads) k_map_scalar(const float *x, float *y, uint64_t n,
                                                         unsigned long long *counters) {
  PHBlock *sh = ph_storage<F>();
  typename F::Regs R;
  F::load(R);
  const int lane = threadIdx.x & 31;
  const uint64_t warp = ((uint64_t)blockIdx.x * kThreads + threadIdx.x) >> 5;
  const uint64_t nwarps = ((uint64_t)gridDim.x * kThreads) >> 5;
  for (uint64_t base = warp * 32; base < n; base += nwarps * 32) {
    uint64_t i = base + lane;
    bool valid = i < n;
    float xs[1] = {valid ? x[i] : 1.0f};
    uint32_t ys[1];
    eval_lanes<F, M, 1>(xs, ys, R, sh, counters);
    if (valid) y[i] = u2f(ys[0]);
  }
}

// sincosf: one reduction, two outputs (1 in / 2 out = 12 B per element).
// The rare mask carries the sin slots in bits 0..15 and the cos slots in
// bits 16..31; one gather pass resolves either kind.
template <int M, int NE, bool STORE_FORM = false>
__device__ __forceinline__ unsigned sincos_lanes(const float (&xs)[NE], uint32_t (&s)[NE],
                                                 uint32_t (&c)[NE], const FnSin::Regs &R,
                                                 PHBlock *sh, unsigned long long *counters) {
  static_assert(NE <= 16, "mask layout");
  RedTrig q[NE];
  trig_reduce<NE>(xs, q, sh);
  unsigned mask = 0;
#pragma unroll
  for (int e = 0; e < NE; ++e) {
    Fast a, b;
    FnSin::sincos_from_red(xs[e], q[e], R, a, b);
    s[e] = f2u(cvt_f32<M>(a.a));
    c[e] = f2u(cvt_f32<M>(b.a));
    rare_or<FnSin>(mask, a.a, xs[e], 1u << e);
    rare_or<FnCos>(mask, b.a, xs[e], 1u << (e + 16));
  }
  if (STORE_FORM) return mask;
  if (__any_sync(kFull, mask != 0)) {
    int cnt = 0;
    do {
      const unsigned low = mask & (0u - mask);
      const unsigned slot = (low | (low >> 16)) & 0xFFFFu;
      const float xe = gather_slot<NE>(xs, slot);
      uint32_t r = 0;
      if (low) r = (low >> 16) ? resolve_one<FnCos, M>(xe, cnt) : resolve_one<FnSin, M>(xe, cnt);
#pragma unroll
      for (int e = 0; e < NE; ++e) {
        s[e] = (low >> e) & 1u ? r : s[e];
        c[e] = (low >> (e + 16)) & 1u ? r : c[e];
      }
      mask &= ~low;
    } while (__any_sync(kFull, mask != 0));
    if (cnt) atomicAdd(counters, (unsigned long long)cnt);
  }
  return 0u;
}

// sincosf takes the store form of the rare path (measured, profiles/r01/ab_rare_store.txt)
constexpr bool kSincosStore = true;

// Store form of the sincosf rare path (after both vector stores): scalar
// overwrite of the one sin or cos output a pending bit names.
template <int M, int NE, int VW>
__device__ __forceinline__ void sincos_rare_store(const float (&xs)[NE], unsigned mask, float *ys,
                                                  float *yc, uint64_t fbase,
                                                  unsigned long long *counters) {
  static_assert(NE <= 16 && (NE & (NE - 1)) == 0, "NE: power of two, <= 16 (16-bit halves)");
  int cnt = 0;
  do {
    const unsigned low = mask & (0u - mask);
    const unsigned slot = (low | (low >> 16)) & 0xFFFFu;
    const float xe = gather_slot<NE>(xs, slot);
    if (low) {
      const uint32_t e = ((uint32_t)__ffs(low) - 1u) & (NE - 1u);
      const uint64_t fi = fbase + (32u * VW * (e / VW) + (e % VW));
      if (low >> 16) yc[fi] = u2f(resolve_one<FnCos, M>(xe, cnt));
      else ys[fi] = u2f(resolve_one<FnSin, M>(xe, cnt));
    }
    mask &= ~low;
  } while (__any_sync(kFull, mask != 0));
  if (cnt) atomicAdd(counters, (unsigned long long)cnt);
}

template <int M, int VW, int NV>
__device__ __forceinline__ void sincos_step(const Vec<VW> *__restrict__ x, Vec<VW> *__restrict__ ys,
                                            Vec<VW> *__restrict__ yc, uint32_t nv, uint32_t base,
                                            uint32_t stride, const Vec<VW> (&cur)[NV],
                                            Vec<VW> (&nxt)[NV], const FnSin::Regs &R, PHBlock *sh,
                                            unsigned long long *counters) {
  float xs[VW * NV];
#pragma unroll
  for (int k = 0; k < NV; ++k) {
    const uint32_t in = base + stride + 32 * k;
    if (in < nv) nxt[k] = ld_vec<VW>(x + in);
#pragma unroll
    for (int j = 0; j < VW; ++j) xs[VW * k + j] = cur[k].v[j];
  }
  uint32_t s[VW * NV], c[VW * NV];
  unsigned mask = sincos_lanes<M, VW * NV, kSincosStore>(xs, s, c, R, sh, counters);
#pragma unroll
  for (int k = 0; k < NV; ++k) {
    const uint32_t i = base + 32 * k;
    if (i < nv) {
      st_vec<VW>(ys + i, s + VW * k);
      st_vec<VW>(yc + i, c + VW * k);
    } else {
      constexpr unsigned kv = (1u << VW) - 1u;
      mask &= ~((kv << (VW * k)) | (kv << (VW * k + 16)));  // stale inputs past the end
    }
  }
  if (kSincosStore && __any_sync(kFull, mask != 0))
    sincos_rare_store<M, VW * NV, VW>(xs, mask, (float *)ys, (float *)yc, (uint64_t)VW * base, counters);
}

#ifndef CRVEC_SINCOS_SHAPE
#define CRVEC_SINCOS_SHAPE 8, 1, 3  // vw, nv, minb (profiles/r01/ab_shtab_trig.txt)
#endif
constexpr int kSincosShape[3] = {CRVEC_SINCOS_SHAPE};
constexpr int kSincosVW = kSincosShape[0], kSincosNV = kSincosShape[1], kSincosMinB = kSincosShape[2];

template <int M>
__global__ void __launch_bounds__(kThreads, kSincosMinB)
    k_sincos_vec(const float *__restrict__ xf, float *__restrict__ ysf, float *__restrict__ ycf,
                 uint32_t nv, unsigned long long *counters) {
  constexpr int VW = kSincosVW, NV = kSincosNV;
  const Vec<VW> *x = reinterpret_cast<const Vec<VW> *>(xf);
  Vec<VW> *ys = reinterpret_cast<Vec<VW> *>(ysf);
  Vec<VW> *yc = reinterpret_cast<Vec<VW> *>(ycf);
  PHBlock *sh = ph_storage<FnSin>();
  FnSin::Regs R;
  FnSin::load(R);
  const uint32_t lane = threadIdx.x & 31;
  const uint32_t stride = gridDim.x * (uint32_t)(kThreads * NV);
  uint32_t base = ((blockIdx.x * kThreads + threadIdx.x) >> 5) * (32 * NV) + lane;
  Vec<VW> va[NV], vb[NV];
#pragma unroll
  for (int k = 0; k < NV; ++k) {
#pragma unroll
    for (int j = 0; j < VW; ++j) va[k].v[j] = 1.f;
    vb[k] = va[k];
    if (base + 32 * k < nv) va[k] = ld_vec<VW>(x + base + 32 * k);
  }
  while (base - lane < nv) {
    sincos_step<M, VW, NV>(x, ys, yc, nv, base, stride, va, vb, R, sh, counters);
    base += stride;
    if (base - lane >= nv) break;
    sincos_step<M, VW, NV>(x, ys, yc, nv, base, stride, vb, va, R, sh, counters);
    base += stride;
  }
}

template <int M>
__global__ void __launch_bounds__(kThreads) k_sincos_scalar(const float *x, float *ys, float *yc,
                                                            uint64_t n, unsigned long long *counters) {
  PHBlock *sh = ph_storage<FnSin>();
  FnSin::Regs R;
  FnSin::load(R);
  const int lane = threadIdx.x & 31;
  const uint64_t warp = ((uint64_t)blockIdx.x * kThreads + threadIdx.x) >> 5;
  const uint64_t nwarps = ((uint64_t)gridDim.x * kThreads) >> 5;
  for (uint64_t base = warp * 32; base < n; base += nwarps * 32) {
    uint64_t i = base + lane;
    bool valid = i < n;
    float xs[1] = {valid ? x[i] : 1.0f};
    uint32_t s[1], c[1];
    sincos_lanes<M, 1>(xs, s, c, R, sh, counters);
    if (valid) {
      ys[i] = u2f(s[0]);
      yc[i] = u2f(c[0]);
    }
  }
}

// ----------------------------------------------------------- sweep kernel ----
__device__ __forceinline__ uint64_t mix64(uint64_t z) {
  z ^= z >> 30;
  z *= 0xbf58476d1ce4e5b9ull;
  z ^= z >> 27;
  z *= 0x94d049bb133111ebull;
  z ^= z >> 31;
  return z;
}

// Per-mode chunk-hash terms mix64((y_m << 32) | p) of one pattern, with two
// mix64 evaluations instead of four: correctly rounded results in the four
// modes take at most two values, RD's and RU's (RZ is one of them, RN is one
// of them), so RN and RZ reuse those hashes. Any other value (never, for
// correct outputs) is still hashed exactly by the fallback branch, so the sum
// stays the definition's whatever the outputs are.
__device__ __forceinline__ void hash4(const uint32_t (&y)[4], uint32_t p, uint64_t *acc) {
  const uint64_t hd = mix64(((uint64_t)y[RD] << 32) | p);
  const uint64_t hu = mix64(((uint64_t)y[RU] << 32) | p);
  uint64_t hn = y[RNE] == y[RD] ? hd : hu;
  uint64_t hz = y[RZ] == y[RD] ? hd : hu;
  if ((y[RNE] != y[RD] && y[RNE] != y[RU]) || (y[RZ] != y[RD] && y[RZ] != y[RU])) {
    hn = mix64(((uint64_t)y[RNE] << 32) | p);
    hz = mix64(((uint64_t)y[RZ] << 32) | p);
  }
  acc[RNE] += hn;
  acc[RZ] += hz;
  acc[RU] += hu;
  acc[RD] += hd;
}

template <class F>
__device__ __forceinline__ void finish4(float x, Fast f, uint32_t (&y)[4], bool &fail) {
  if constexpr (HasTiny<F>::value) {
    const uint32_t xb = f2u(x);
    if (f.main && F::is_tiny(xb)) {  // the map kernels' result-bits rule
      fail = false;
      y[0] = F::template tiny_bits<RNE>(xb);
      y[1] = F::template tiny_bits<RZ>(xb);
      y[2] = F::template tiny_bits<RU>(xb);
      y[3] = F::template tiny_bits<RD>(xb);
      return;
    }
  }
  if (f.main) {
    y[0] = finish<RNE>(f, fail, F::E);
    bool d;
    y[1] = finish<RZ>(f, d, F::E);
    y[2] = finish<RU>(f, d, F::E);
    y[3] = finish<RD>(f, d, F::E);
  } else {
    fail = false;
    y[0] = F::template special<RNE>(x);
    y[1] = F::template special<RZ>(x);
    y[2] = F::template special<RU>(x);
    y[3] = F::template special<RD>(x);
  }
}
__device__ __forceinline__ void round4(DD v, uint32_t (&y)[4]) {
  y[0] = round_dd<RNE>(v.hi, v.lo);
  y[1] = round_dd<RZ>(v.hi, v.lo);
  y[2] = round_dd<RU>(v.hi, v.lo);
  y[3] = round_dd<RD>(v.hi, v.lo);
}

// Block-wide sum of 4 (or 8) u64 lanes into global accumulators.
template <int K>
__device__ __forceinline__ void block_add(uint64_t (&acc)[K], uint64_t *dst) {
  __shared__ uint64_t red[kWarps][K];
#pragma unroll
  for (int m = 0; m < K; ++m)
    for (int o = 16; o; o >>= 1) acc[m] += __shfl_xor_sync(kFull, acc[m], o);
  if ((threadIdx.x & 31) == 0)
#pragma unroll
    for (int m = 0; m < K; ++m) red[threadIdx.x >> 5][m] = acc[m];
  __syncthreads();
  if (threadIdx.x < K) {
    uint64_t s = 0;
    for (int w = 0; w < kWarps; ++w) s += red[w][threadIdx.x];
    atomicAdd((unsigned long long *)&dst[threadIdx.x], (unsigned long long)s);
  }
}

// Exhaustive sweep over binary32 patterns: each block covers 4096 patterns of
// one 2^20 chunk (256 blocks per chunk); every pattern is evaluated once and
// converted in all four modes; per chunk and mode the hashes are summed.
constexpr int kSweepPerThread = 64;
constexpr int kSweepPerBlock = kThreads * kSweepPerThread;  // 16384 (64 per thread: 0.348 -> 0.323 s, tools/sweep_time.py)
constexpr int kSweepBlocksPerChunk = (1 << 20) / kSweepPerBlock;

template <class F, bool FORCE>
__global__ void __launch_bounds__(kThreads) k_sweep(uint32_t chunk_lo, uint64_t *hashes,
                                                    unsigned long long *counters) {
  PHBlock *sh = ph_storage<F>();
  typename F::Regs R;
  F::load(R);
  uint32_t chunk = chunk_lo + blockIdx.x / kSweepBlocksPerChunk;
  uint32_t p0 = (chunk << 20) + (blockIdx.x % kSweepBlocksPerChunk) * kSweepPerBlock;
  uint64_t acc[4] = {0, 0, 0, 0};
  int nslow = 0;
#pragma unroll 1
  for (int it = 0; it < kSweepPerThread / 4; ++it) {
    uint32_t pb = p0 + it * (kThreads * 4) + threadIdx.x * 4;
    float xs[4];
#pragma unroll
    for (int e = 0; e < 4; ++e) xs[e] = u2f(pb + e);
    Fast f[4];
    fast_lanes<F, 4>(xs, f, R, sh);
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      uint32_t y[4];
      bool fail;
      uint32_t xb = pb + e;
      finish4<F>(xs[e], f[e], y, fail);
      if (fail || (FORCE && f[e].main)) {
        round4(slow_dd<F>(xs[e]), y);
        ++nslow;
      }
      hash4(y, xb, acc);
    }
  }
  if (nslow) atomicAdd(counters, (unsigned long long)nslow);
  block_add<4>(acc, hashes + 4ull * (chunk - chunk_lo));
}

template <bool FORCE>
__global__ void __launch_bounds__(kThreads) k_sweep_sincos(uint32_t chunk_lo, uint64_t *hs,
                                                           uint64_t *hc,
                                                           unsigned long long *counters) {
  PHBlock *sh = ph_storage<FnSin>();
  FnSin::Regs R;
  FnSin::load(R);
  uint32_t chunk = chunk_lo + blockIdx.x / kSweepBlocksPerChunk;
  uint32_t p0 = (chunk << 20) + (blockIdx.x % kSweepBlocksPerChunk) * kSweepPerBlock;
  uint64_t acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  int nslow = 0;
#pragma unroll 1
  for (int it = 0; it < kSweepPerThread / 4; ++it) {
    uint32_t pb = p0 + it * (kThreads * 4) + threadIdx.x * 4;
    float xs[4];
    RedTrig q[4];
#pragma unroll
    for (int e = 0; e < 4; ++e) xs[e] = u2f(pb + e);
    trig_reduce<4>(xs, q, sh);
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      uint32_t xb = pb + e;
      Fast a, b;
      FnSin::sincos_from_red(xs[e], q[e], R, a, b);
      uint32_t ys[4], yc[4];
      bool fs, fc;
      finish4<FnSin>(xs[e], a, ys, fs);
      finish4<FnCos>(xs[e], b, yc, fc);
      if (fs || (FORCE && a.main)) { round4(slow_dd<FnSin>(xs[e]), ys); ++nslow; }
      if (fc || (FORCE && b.main)) { round4(slow_dd<FnCos>(xs[e]), yc); ++nslow; }
      hash4(ys, xb, acc);
      hash4(yc, xb, acc + 4);
    }
  }
  if (nslow) atomicAdd(counters, (unsigned long long)nslow);
  uint64_t a4[4] = {acc[0], acc[1], acc[2], acc[3]};
  uint64_t c4[4] = {acc[4], acc[5], acc[6], acc[7]};
  block_add<4>(a4, hs + 4ull * (chunk - chunk_lo));
  __syncthreads();
  block_add<4>(c4, hc + 4ull * (chunk - chunk_lo));
}


// ------------------------------------------------------- hard-case screen ----
// GPU worst-case finder (the reference's hardest_case_search,
// ref: proj/src/oracle.cpp:565-580, is a CPU loop over MPFR): every pattern of
// the chunk range is evaluated on the double-double path and its relative
// distance to the nearest binary32 rounding boundary (representable value or
// midpoint, any mode) is measured; inputs closer than 2^-thr are appended.
__device__ __forceinline__ double boundary_rel_distance(DD v) {
  double h = v.hi;
  if (!(dabs(h) < 0x1p128) || h == 0.0) return 1.0;
  uint64_t b = d2u(h);
  uint64_t q = (b + (1ull << 27)) & ~((1ull << 28) - 1);  // nearest 25-bit lattice point
  double dq = u2d(q);
  double d = add_(sub_(h, dq), v.lo);  // h - dq exact (same or adjacent binade)
  return dabs(d) / dabs(h);
}

template <class F>
__global__ void __launch_bounds__(kThreads) k_hardscan(uint32_t chunk_lo, double thr,
                                                       uint32_t *out_bits, double *out_dist,
                                                       unsigned long long cap,
                                                       unsigned long long *count) {
  typename F::Regs R;
  F::load(R);
  uint32_t chunk = chunk_lo + blockIdx.x / kSweepBlocksPerChunk;
  uint32_t p0 = (chunk << 20) + (blockIdx.x % kSweepBlocksPerChunk) * kSweepPerBlock;
#pragma unroll 1
  for (int it = 0; it < kSweepPerThread; ++it) {
    uint32_t xb = p0 + it * kThreads + threadIdx.x;
    float x = u2f(xb);
    Fast f;
    if constexpr (IsTrig<F>::value) f = F::from_red(x, RedTrig{0, 0.0}, R);  // only .main is used
    else f = F::fast(x, R);
    if (f.main && F::in_main(xb)) {  // divergent body without shuffles; fast() above runs converged
      double d = boundary_rel_distance(slow_dd<F>(x));
      if (d < thr) {
        unsigned long long k = atomicAdd(count, 1ull);
        if (k < cap) {
          out_bits[k] = xb;
          out_dist[k] = d;
        }
      }
    }
    __syncwarp();
  }
}

template <class F>
cudaError_t launch_hardscan(uint32_t chunk_lo, uint32_t chunk_hi, double thr, uint32_t *bits,
                            double *dist, unsigned long long cap, unsigned long long *count,
                            cudaStream_t s) {
  unsigned blocks = (chunk_hi - chunk_lo) * kSweepBlocksPerChunk;
  k_hardscan<F><<<blocks, kThreads, 0, s>>>(chunk_lo, thr, bits, dist, cap, count);
  return cudaGetLastError();
}

// ------------------------------------------------------------- launchers ----
using MapLaunch = cudaError_t (*)(const float *, float *, float *, uint64_t, cudaStream_t,
                                  unsigned long long *);
using SweepLaunch = cudaError_t (*)(uint32_t, uint32_t, uint64_t *, uint64_t *, int, cudaStream_t,
                                    unsigned long long *);

template <class K>
inline int max_blocks(K kernel) {
  int dev = 0, sms = 148, per = 1;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, kernel, kThreads, 0);
  if (per < 1) per = 1;
  return sms * per;
}

// Vectors per launch of the map kernels: they index vectors with 32 bits, so
// a launch covers at most 2^31 vectors. CRVEC_SPLIT_VECTORS (read once) lowers
// the split point so the tests can exercise multi-launch calls at small sizes.
inline uint64_t max_vectors_per_launch() {
  static const uint64_t v = [] {
    const char *e = getenv("CRVEC_SPLIT_VECTORS");
    unsigned long long k = e ? strtoull(e, nullptr, 10) : 0ull;
    return (k >= 32 && k < (1ull << 31)) ? (uint64_t)k : (uint64_t(1) << 31);
  }();
  return v;
}

inline unsigned grid_for(uint64_t work_warps32, int maxb) {
  // work_warps32 = number of 32-lane slots; one warp per slot per pass
  uint64_t blocks = (work_warps32 + kWarps - 1) / kWarps;
  if (blocks > 4ull * (uint64_t)maxb) blocks = 4ull * (uint64_t)maxb;  // 4 waves: better tail balance
  return (unsigned)(blocks ? blocks : 1);
}

template <class F, int M>
cudaError_t launch_map(const float *x, float *y, float *, uint64_t n, cudaStream_t s,
                       unsigned long long *ctr) {
  constexpr int VW = KernelShape<F>::vw, NV = KernelShape<F>::nv;
  static int mb_vec = max_blocks(k_map_vec<F, M>);
  static int mb_sc = max_blocks(k_map_scalar<F, M>);
  constexpr uintptr_t A = 4 * VW - 1;  // vector alignment mask (16 or 32 bytes)
  auto scalar = [&](const float *xx, float *yy, uint64_t m) {
    if (m) k_map_scalar<F, M><<<grid_for((m + 31) / 32, mb_sc), kThreads, 0, s>>>(xx, yy, m, ctr);
  };
  // x and y misaligned by the same amount: peel a scalar head up to the
  // vector boundary (a relative misalignment leaves only the element kernel)
  uint64_t head = 0;
  if ((((uintptr_t)x ^ (uintptr_t)y) & A) == 0 && ((uintptr_t)x & 3) == 0 && ((uintptr_t)x & A))
    head = ((A + 1 - ((uintptr_t)x & A)) & A) / 4;
  if (head > n) head = n;
  const bool aligned = ((((uintptr_t)(x + head)) | ((uintptr_t)(y + head))) & A) == 0;
  const uint64_t nvec = aligned ? (n - head) / VW : 0;
  scalar(x, y, aligned ? head : 0);
  const float *xv = aligned ? x + head : x;
  float *yv = aligned ? y + head : y;
  // the kernel indexes vectors with 32 bits: launches of at most 2^31 vectors
  const uint64_t kMaxNV = max_vectors_per_launch();
  for (uint64_t off = 0; off < nvec; off += kMaxNV) {
    uint64_t m = nvec - off < kMaxNV ? nvec - off : kMaxNV;
    const unsigned g = grid_for((m + 32 * NV - 1) / (32 * NV), mb_vec);
    k_map_vec<F, M><<<g, kThreads, 0, s>>>(xv + VW * off, yv + VW * off, (uint32_t)m, ctr);
  }
  scalar(xv + VW * nvec, yv + VW * nvec, (uint64_t)((x + n) - (xv + VW * nvec)));
  return cudaGetLastError();
}

template <int M>
cudaError_t launch_sincos(const float *x, float *ys, float *yc, uint64_t n, cudaStream_t s,
                          unsigned long long *ctr) {
  constexpr int VW = kSincosVW, NV = kSincosNV;
  static int mb_vec = max_blocks(k_sincos_vec<M>);
  static int mb_sc = max_blocks(k_sincos_scalar<M>);
  constexpr uintptr_t A = 4 * VW - 1;
  auto scalar = [&](uint64_t off, uint64_t m) {
    if (m)
      k_sincos_scalar<M><<<grid_for((m + 31) / 32, mb_sc), kThreads, 0, s>>>(x + off, ys + off, yc + off,
                                                                               m, ctr);
  };
  // the three arrays equally misaligned: peel a scalar head to the vector boundary
  uint64_t head = 0;
  const uintptr_t ax = (uintptr_t)x & A;
  if (((uintptr_t)ys & A) == ax && ((uintptr_t)yc & A) == ax && (ax & 3) == 0 && ax)
    head = ((A + 1 - ax) & A) / 4;
  if (head > n) head = n;
  const bool aligned = ((((uintptr_t)(x + head)) | ((uintptr_t)(ys + head)) | ((uintptr_t)(yc + head))) & A) == 0;
  const uint64_t nvec = aligned ? (n - head) / VW : 0;
  const uint64_t v0 = aligned ? head : 0;
  scalar(0, v0);
  const uint64_t kMaxNV = max_vectors_per_launch();
  for (uint64_t off = 0; off < nvec; off += kMaxNV) {
    uint64_t m = nvec - off < kMaxNV ? nvec - off : kMaxNV;
    const uint64_t f = v0 + VW * off;
    k_sincos_vec<M><<<grid_for((m + 32 * NV - 1) / (32 * NV), mb_vec), kThreads, 0, s>>>(
        x + f, ys + f, yc + f, (uint32_t)m, ctr);
  }
  scalar(v0 + VW * nvec, n - (v0 + VW * nvec));
  return cudaGetLastError();
}

template <class F>
cudaError_t launch_sweep(uint32_t chunk_lo, uint32_t chunk_hi, uint64_t *h, uint64_t *, int force,
                         cudaStream_t s, unsigned long long *ctr) {
  unsigned blocks = (chunk_hi - chunk_lo) * kSweepBlocksPerChunk;
  if (force) k_sweep<F, true><<<blocks, kThreads, 0, s>>>(chunk_lo, h, ctr);
  else k_sweep<F, false><<<blocks, kThreads, 0, s>>>(chunk_lo, h, ctr);
  return cudaGetLastError();
}

inline cudaError_t launch_sweep_sincos(uint32_t chunk_lo, uint32_t chunk_hi, uint64_t *h,
                                       uint64_t *h2, int force, cudaStream_t s,
                                       unsigned long long *ctr) {
  unsigned blocks = (chunk_hi - chunk_lo) * kSweepBlocksPerChunk;
  if (force) k_sweep_sincos<true><<<blocks, kThreads, 0, s>>>(chunk_lo, h, h2, ctr);
  else k_sweep_sincos<false><<<blocks, kThreads, 0, s>>>(chunk_lo, h, h2, ctr);
  return cudaGetLastError();
}

// Registration: each family translation unit fills its rows.
using ScanLaunch = cudaError_t (*)(uint32_t, uint32_t, double, uint32_t *, double *,
                                   unsigned long long, unsigned long long *, cudaStream_t);
struct FnEntry {
  MapLaunch map[4];
  SweepLaunch sweep;
  ScanLaunch scan;
};
template <class F>
constexpr FnEntry make_entry() {
  return FnEntry{{launch_map<F, RNE>, launch_map<F, RZ>, launch_map<F, RU>, launch_map<F, RD>},
                 launch_sweep<F>, launch_hardscan<F>};
}

}  // namespace crvec
