# end-to-end (pht_pc_step_host) A/B of libraries: bench.py's step + e2e only, twice each
L=$PWD/paper_2111_14317_b200
for i in 1 2; do for v in "$@"; do
  PHT_LIB=$L/$v/libpht.so python bench.py --tracking "" --no-evaluation --no-paper-protocol --no-cpu-baseline 2>/dev/null | tail -1 | python -c "
import sys,json; d=json.load(sys.stdin); print('$v', round(d['value']/1e6,1), round(d['e2e']['value']/1e6,1), [round(x/5,2) for x in d['e2e']['runs_ms']], round(d['e2e']['link_ms_per_step'],2))"
done; done > gpurun_out/e2e_ab.txt
