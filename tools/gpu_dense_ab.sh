# A/B of the DMMA evaluation kernel: tools/dense_bench.py on lib vs lib_old, then the dense parity tests
L=$PWD/paper_2111_14317_b200
for i in 1 2; do for v in lib lib_old; do echo "$v $(PHT_LIB=$L/$v/libpht.so python tools/dense_bench.py 2>&1 | tail -1)"; done; done > gpurun_out/dab.txt
python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "dense or ragged or rescale or round_trip" > gpurun_out/t_dense.log 2>&1
if [ "$1" == "ncu" ]; then PHT_REPS=1 timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_dense -s 2 -c 1 -o gpurun_out/dense_lib python tools/dense_bench.py > gpurun_out/ncu_lib.log 2>&1; fi
