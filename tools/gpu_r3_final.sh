# Final evidence on one B200: GPU tests, smoke, the default bench line, the launch list of a short
# bench, ncu --set full of the evaluation (k_evalw, cyclic-10) and of the tracker (k_trackw, cyclic-10).
mkdir -p gpurun_out
python -m pytest tests -m gpu -q > gpurun_out/gpu_tests.log 2>&1; echo "rc=$?" >> gpurun_out/gpu_tests.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "rc=$?" >> gpurun_out/smoke.log
python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_evalw -s 1 -c 1 -f \
    -o gpurun_out/evalw_final python tools/eval_once.py > gpurun_out/ncu_evalw.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_trackw -s 1 -c 1 -f \
    -o gpurun_out/trk_final python tools/track_bench.py cyclic-10:1000000 > gpurun_out/ncu_trk.log 2>&1
