#!/bin/bash
# katsura-10 tracking (990 paths, time to the last path) per library, 3 runs each
L=$PWD/paper_2111_14317_b200
for v in "$@"; do
  for r in 1 2 3; do
    echo "$v $(PHT_LIB=$L/$v/libpht.so python tools/track_bench.py katsura-10:10000 2>&1 | grep '^{' | python -c 'import json,sys; d=json.loads(sys.stdin.read()); k=list(d)[0]; print(round(d[k]["ms"],2), d[k]["status"][0])')"
  done
done
