# Final evidence on one B200: GPU tests, smoke, the default bench line, the launch list of the bench
# command, and ncu --set full of the C4 DMMA evaluation (k_dense<20>).
mkdir -p gpurun_out
python -m pytest tests -m gpu -q > gpurun_out/gpu_tests.log 2>&1; echo "rc=$?" >> gpurun_out/gpu_tests.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "rc=$?" >> gpurun_out/smoke.log
python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv \
    python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/ncu_launch.log 2>&1
PHT_REPS=1 timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_dense -s 2 -c 1 -f \
    -o gpurun_out/dense_final python tools/dense_bench.py > gpurun_out/ncu_dense.log 2>&1
