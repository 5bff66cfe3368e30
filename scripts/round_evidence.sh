#!/bin/bash
# Round-end evidence on one B200 (gpurun): GPU suite, smoke, bench (own arm + reference arm), one
# bench line per config, the launch list of one bench step, and ncu --set full captures of the
# PCG SpMV and the numeric assembly.  Everything lands in gpurun_out/$TAG/.
TAG=${TAG:-r02z}
O=gpurun_out/$TAG
mkdir -p $O
export PYTHONUNBUFFERED=1
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $O/gpu.txt
timeout 1500 python -m pytest tests -m gpu -q > $O/pytest_gpu.log 2>&1; tail -1 $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; tail -1 $O/smoke.log
timeout 900 python bench.py > $O/bench.json 2> $O/bench.err; tail -c 300 $O/bench.json
timeout 900 python bench.py --impl reference --steps 1 --warmup 3 > $O/reference_arm.json 2> $O/reference_arm.err
mkdir -p $O/all_configs
for c in 1 2 3 4 5; do
  timeout 900 python bench.py --config $c --steps 2 --warmup 3 --no-cpu-baseline \
    > $O/all_configs/bench_cfg$c.json 2> $O/all_configs/bench_cfg$c.err || echo "cfg$c failed"
done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 4000 --csv --log-file $O/launches_bench_cfg4.csv \
  python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-e2e > $O/launches_bench.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_spmv_df -s 5 -c 1 -o $O/df \
  python scripts/profile_step.py --config 4 --pcg-iters 8 > $O/ncu_df.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_asm_tile -s 1 -c 1 -o $O/asm \
  python scripts/profile_step.py --config 4 --pcg-iters 2 --reassemble 2 > $O/ncu_asm.log 2>&1
ls -la $O
