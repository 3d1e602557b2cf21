set -x
python -m pytest tests -m gpu -q 2>&1 | tail -30 > gpurun_out/gpu_tests.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
python bench.py --steps 10 --warmup 3 > gpurun_out/bench.json 2> gpurun_out/bench.err
ncu --metrics gpu__time_duration.sum --clock-control none -c 20 --csv --log-file gpurun_out/launches.csv python bench.py --steps 3 --warmup 3 --points 1048576 --no-cpu-baseline --e2e-steps 1 > gpurun_out/ncu_launch.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_pht -s 3 -c 1 -o gpurun_out/prof_step python bench.py --steps 2 --warmup 3 --points 262144 --no-cpu-baseline --e2e-steps 1 > gpurun_out/ncu_full.log 2>&1
ls -la gpurun_out
