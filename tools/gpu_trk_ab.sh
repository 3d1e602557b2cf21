# tracker A/B of libraries: noon-10 and cyclic-10 (all paths), three alternating rounds
L=$PWD/paper_2111_14317_b200
for i in 1 2 3; do for v in "$@"; do
  PHT_LIB=$L/$v/libpht.so python tools/track_bench.py noon-10:10000 cyclic-10:1000000 2>/dev/null | python -c "
import sys,json
r={}
for l in sys.stdin:
    if l.startswith('{'):
        d=json.loads(l); k=list(d)[0]; r[k.split(':')[0]]=(round(d[k]['ms'],2), d[k]['status'][0])
print('$v', r)"
done; done > gpurun_out/trk_ab.txt
