#!/bin/bash
# parity tests touched by the rescale fix, then k_stepw compile-time variants (pc_step M evals/s)
mkdir -p gpurun_out
python -m pytest tests/test_gpu_parity.py -q -p no:cacheprovider -k "range_stress or extreme_rows or rescale or dense_tensor" 2>&1 | tail -4
L=$PWD/paper_2111_14317_b200
for v in lib "$@"; do
  echo "$v $(PHT_LIB=$L/$v/libpht.so python tools/step_bench.py 2>&1 | tail -1)"
done
