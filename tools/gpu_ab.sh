# A/B of kernel variants: parity tests on the default build, bench on each variant.
set -x
python -m pytest tests -m gpu -q -x 2>&1 | tail -5 > gpurun_out/gpu_tests.log
for v in lib lib_pts16; do
  PHT_LIB=$PWD/paper_2111_14317_b200/$v/libpht.so python bench.py --steps 10 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/bench_$v.json 2>gpurun_out/bench_$v.err
done
