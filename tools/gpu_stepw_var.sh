# compile-time variants of the warp-per-group kernels: pc_step throughput and tracking times
mkdir -p gpurun_out
L=$PWD/paper_2111_14317_b200
rm -f gpurun_out/swv.txt
for v in "$@"; do
  PHT_LIB=$L/$v/libpht.so python tools/step_bench.py > gpurun_out/swv_$v.txt 2>&1; echo "$v $(tail -1 gpurun_out/swv_$v.txt)" >> gpurun_out/swv.txt
  PHT_LIB=$L/$v/libpht.so python tools/track_bench.py katsura-10:10000 noon-10:10000 cyclic-10:1000000 > gpurun_out/swt_$v.txt 2>&1
  echo "$v $(python -c "
import json
r={}
for l in open('gpurun_out/swt_$v.txt'):
    if l.startswith('{'):
        d=json.loads(l); k=list(d)[0]; r[k.split(':')[0]]=round(d[k]['ms'],1)
print(r)")" >> gpurun_out/swv.txt
done
