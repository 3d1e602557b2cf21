mkdir -p gpurun_out
python -m pytest tests/test_gpu_track.py -q -x > gpurun_out/trk_tests.log 2>&1; echo "rc=$?" >> gpurun_out/trk_tests.log
rm -f gpurun_out/herm.txt
for o in '{}' '{"predictor": 1}'; do
  echo "$o" >> gpurun_out/herm.txt
  TB_OPTS="$o" python tools/track_bench.py katsura-10:10000 noon-10:10000 cyclic-10:1000000 >> gpurun_out/herm.txt 2>&1
done
