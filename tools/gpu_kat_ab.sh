# katsura-10 tracking (time to the last path) A/B of libraries, 4 alternating rounds
L=$PWD/paper_2111_14317_b200
for i in 1 2 3 4; do for v in "$@"; do
  PHT_LIB=$L/$v/libpht.so python tools/track_bench.py katsura-10:10000 2>/dev/null | python -c "
import sys,json
for l in sys.stdin:
    if l.startswith('{'):
        d=json.loads(l); k=list(d)[0]; print('$v', round(d[k]['ms'],3), d[k]['status'][0])"
done; done > gpurun_out/kat_ab.txt
