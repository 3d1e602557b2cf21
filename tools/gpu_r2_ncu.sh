#!/bin/bash
# ncu --set full of one k_stepw<10, STEP> launch (cyclic-10, 2^20 points) per library
mkdir -p gpurun_out
L=$PWD/paper_2111_14317_b200
for v in "$@"; do
  PHT_LIB=$L/$v/libpht.so ncu --set full --clock-control none --import-source on -k regex:k_stepw -s 1 -c 1 \
      -o gpurun_out/r02_step_$v -f python tools/step_once.py > gpurun_out/ncu_$v.log 2>&1
  echo "$v rc=$?"
done
