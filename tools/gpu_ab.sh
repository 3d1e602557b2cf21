python -m pytest tests -m gpu -q 2>&1 | tail -8 > gpurun_out/gpu_tests.log
python tools/track_bench.py katsura-10:10000 noon-10:10000 cyclic-10:1000000 > gpurun_out/tb_plog.json 2>/dev/null
TB_OPTS='{"newton_tol": 1e-8}' python tools/track_bench.py katsura-10:10000 noon-10:10000 cyclic-10:1000000 > gpurun_out/tb_plog_tol8.json 2>/dev/null
