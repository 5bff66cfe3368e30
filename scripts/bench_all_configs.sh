#!/bin/bash
# One bench line per BASELINE config (cfg1-5, FS-FEM) on one GPU; results to gpurun_out/bench_cfg*.json.
for c in 1 2 3 4 5; do
  timeout 900 python bench.py --config $c --steps ${STEPS:-2} --warmup ${WARMUP:-3} --no-cpu-baseline \
    > gpurun_out/bench_cfg$c.json 2> gpurun_out/bench_cfg$c.err || echo "cfg$c failed"
done
