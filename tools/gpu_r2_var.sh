#!/bin/bash
# k_stepw / k_trackw compile-time variants: pc_step M evals/s and tracking ms per library
mkdir -p gpurun_out
L=$PWD/paper_2111_14317_b200
for v in "$@"; do
  echo "$v step $(PHT_LIB=$L/$v/libpht.so python tools/step_bench.py 2>&1 | tail -1)"
  PHT_LIB=$L/$v/libpht.so python tools/track_bench.py katsura-10:10000 noon-10:10000 cyclic-10:1000000 > gpurun_out/swt_$v.txt 2>&1
  echo "$v track $(python -c "
import json
r={}
for l in open('gpurun_out/swt_$v.txt'):
    if l.startswith('{'):
        d=json.loads(l); k=list(d)[0]; r[k.split(':')[0]]=(round(d[k]['ms'],2), d[k].get('status'))
print(r)")"
done
