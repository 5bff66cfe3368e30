#!/bin/bash
# Time the PCG SpMV of each tuning build (build/libfsfem_*.so) and the product library on cfg4.
for lib in paper_2001_08849_b200/libfsfem.so build/libfsfem_*.so; do
  echo "== $lib"
  FSFEM_LIB=$lib python scripts/profile_step.py --config ${1:-4} --pcg-iters 128 --reassemble 1 2>&1 | tail -1
done
