# k_evalu (records as a kernel parameter) vs k_evalw (records in shared memory): pht_evaluate throughput
L=$PWD/paper_2111_14317_b200
for i in 1 2; do for v in "$@"; do echo "$v $(PHT_LIB=$L/$v/libpht.so python tools/eval_ab.py lane 2>&1 | tail -1)"; done; done > gpurun_out/evalu_ab.txt
