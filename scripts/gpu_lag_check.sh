# Lagged push SpMV (k_spmv_lag) vs the dataflow kernel: parity of the lag kernel, then cfg4 SpMV
# per-call times of the product library and the tuning builds in build/.
set -x
export PYTHONUNBUFFERED=1
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1200 python -m pytest tests/test_gpu_spmv_kernels.py -x -q -k "lag and cfg3" 2>&1 | tail -3
for lib in paper_2001_08849_b200/libfsfem.so build/libfsfem_*.so; do
  for k in ${KERNELS:-dataflow lag}; do
    echo "== $lib $k"; FSFEM_LIB=$lib FSFEM_SPMV_KERNEL=$k timeout 300 python scripts/spmv_bench.py --config 4 --reps 200 2>&1 | tail -1
  done
done
