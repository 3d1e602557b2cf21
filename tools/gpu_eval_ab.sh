# Standalone evaluation throughput: DMMA path, generic W-layout kernel, specialised kernels; parity.
mkdir -p gpurun_out
PHT_DENSE=1 python tools/eval_bench.py > gpurun_out/ev_dense.txt 2>&1
PHT_DENSE=0 python tools/eval_bench.py > gpurun_out/ev_generic.txt 2>&1
PHT_SPEC=1 python tools/eval_bench.py > gpurun_out/ev_spec.txt 2>&1
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_specialized.py -q -x > gpurun_out/ev_par.log 2>&1; echo "rc=$?" >> gpurun_out/ev_par.log
