# ncu --set full (source-level) of the katsura-10 tracker launch (k_trackw, LPR = 2) + a timing run
python tools/track_bench.py katsura-10:10000 > gpurun_out/trk_kat.json 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_trackw -s 1 -c 1 -o gpurun_out/trk_kat python tools/track_bench.py katsura-10:10000 > gpurun_out/ncu_trk.log 2>&1
