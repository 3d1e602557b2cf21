# A/B of the warp-per-group tracker (PHT_TRACKW=1, default) vs the tile tracker (PHT_TRACKW=0).
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_track.py tests/test_gpu_param.py tests/test_gpu_fullsize.py tests/test_gpu_specialized.py tests/test_gpu_edges.py -q -x > gpurun_out/tw_tests.log 2>&1; echo "rc=$?" >> gpurun_out/tw_tests.log
for rep in 1 2 3; do
for m in 0 1; do
  PHT_TRACKW=$m python tools/track_bench.py katsura-10:10000 noon-10:10000 cyclic-10:1000000 > gpurun_out/tw_track_${m}_$rep.txt 2>&1
done
done
