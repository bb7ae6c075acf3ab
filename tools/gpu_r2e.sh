#!/bin/bash
# round-2 bench refresh (reference arm with the generated tables linked; sweep warm-up) + PCIe ceiling probe
O=gpurun_out/r2e; mkdir -p $O
nvidia-smi topo -m > $O/topo.txt 2>&1; nvidia-smi -q | grep -i -A3 "PCI\b\|Link Width\|Link Gen\|Max Link" > $O/pcie.txt 2>&1
timeout 900 python bench.py --steps 10 --warmup 3 > $O/bench.json 2> $O/bench.err; tail -c 300 $O/bench.json
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > $O/bench_ref.json 2> $O/bench_ref.err; cat $O/bench_ref.json | head -c 600
timeout 300 python tools/e2e_probe.py > $O/e2e_probe.txt 2>&1; cat $O/e2e_probe.txt
