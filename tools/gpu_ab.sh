TB_OPTS='{"dtau_min": 1e-12}' python tools/track_bench.py katsura-10:10000 noon-10:10000 cyclic-10:1000000 > gpurun_out/tb_min12.json 2>/dev/null
TB_OPTS='{"dtau_min": 1e-14, "max_steps": 100000}' python tools/track_bench.py katsura-10:10000 noon-10:10000 cyclic-10:1000000 > gpurun_out/tb_min14.json 2>/dev/null
TB_OPTS='{"dtau_min": 1e-12, "newton_tol": 1e-8}' python tools/track_bench.py katsura-10:10000 noon-10:10000 cyclic-10:1000000 > gpurun_out/tb_min12_tol8.json 2>/dev/null
