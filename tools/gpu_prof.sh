# ncu captures of the pc_step kernel: generic and system-specialised (cyclic-10)
mkdir -p gpurun_out
ncu --set full --clock-control none --import-source on -k regex:k_pht -s 1 -c 1 -o gpurun_out/prof_step_gen python tools/step_once.py > gpurun_out/ncu_gen.log 2>&1
PHT_SPEC=1 ncu --set full --clock-control none --import-source on -k regex:k_pht -s 1 -c 1 -o gpurun_out/prof_step_jit python tools/step_once.py > gpurun_out/ncu_jit.log 2>&1
