mkdir -p gpurun_out
python -m pytest tests -m gpu -q -x > gpurun_out/ab_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/ab_tests.log
python tools/jit_check.py > gpurun_out/jit_check.txt 2>&1
PHT_SPEC=1 python tools/track_bench.py katsura-10:10000 noon-10:10000 cyclic-10:1000000 > gpurun_out/jit_track.txt 2>&1
PHT_SPEC=1 python tools/eval_bench.py > gpurun_out/jit_eval.txt 2>&1
