# k_dense compile-time variants (tools/variant_n10.sh <name> "<flags>" 20): C4 throughput per library
L=$PWD/paper_2111_14317_b200
for i in 1 2; do for v in "$@"; do echo "$v $(PHT_LIB=$L/$v/libpht.so python tools/dense_bench.py 2>&1 | tail -1)"; done; done > gpurun_out/dvar.txt
