#!/bin/bash
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -q -m gpu 2>&1 | tail -30 > gpurun_out/pytest6.txt
timeout 300 python bench.py > gpurun_out/bench6.json 2> gpurun_out/bench6.err
timeout 300 python bench.py --impl reference --steps 5 --warmup 1 > gpurun_out/bench6_ref.json 2>&1
