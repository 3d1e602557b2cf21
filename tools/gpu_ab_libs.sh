# A/B of whole libraries: step throughput, tracking times (3 configs), evaluation (lane family), twice each
mkdir -p gpurun_out
L=$PWD/paper_2111_14317_b200
rm -f gpurun_out/ab.txt
for r in 1 2; do for v in "$@"; do
  echo "$v step $(PHT_LIB=$L/$v/libpht.so python tools/step_bench.py 2>&1 | tail -1)" >> gpurun_out/ab.txt
  PHT_LIB=$L/$v/libpht.so python tools/track_bench.py katsura-10:10000 noon-10:10000 cyclic-10:1000000 > gpurun_out/abt_$v.txt 2>&1
  echo "$v track $(python -c "
import json
r={}
for l in open('gpurun_out/abt_$v.txt'):
    if l.startswith('{'):
        d=json.loads(l); k=list(d)[0]; r[k.split(':')[0]]=(round(d[k]['ms'],2), d[k]['status'][0])
print(r)")" >> gpurun_out/ab.txt
  echo "$v eval $(PHT_LIB=$L/$v/libpht.so python tools/eval_ab.py lane 2>&1 | tail -1)" >> gpurun_out/ab.txt
done; done
