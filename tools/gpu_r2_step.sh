#!/bin/bash
# pc_step throughput per library (tools/step_bench.py)
L=$PWD/paper_2111_14317_b200
for v in "$@"; do echo "$v $(PHT_LIB=$L/$v/libpht.so python tools/step_bench.py 2>&1 | tail -1)"; done
