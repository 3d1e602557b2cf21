# ncu --set full (source-level) of one tracker launch (k_trackw) per config: tools/gpu_trk_prof.sh katsura-10:10000 cyclic-10:1000000
mkdir -p gpurun_out
for c in "$@"; do
  n=${c%%:*}
  python tools/track_bench.py $c > gpurun_out/trk_$n.json 2>&1
  timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_trackw -s 1 -c 1 -f -o gpurun_out/trk_$n python tools/track_bench.py $c > gpurun_out/ncu_trk_$n.log 2>&1
done
