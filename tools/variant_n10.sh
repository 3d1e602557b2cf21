#!/bin/bash
# Fast compile-time variant of the n = 10 (and optionally n = 11) kernels: compile those translation
# units with extra flags and link them with the main build's other objects into lib_<name>/libpht.so.
#   tools/variant_n10.sh <name> "<nvcc flags>" [ns...]
set -e
name=$1; flags=$2; shift 2; ns=${@:-10}
C=$(dirname $0)/../paper_2111_14317_b200/csrc
cd $C
NV="/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -Xcompiler -O2 --expt-relaxed-constexpr"
mkdir -p build_var/$name ../lib_$name
objs=""
for o in build/*.o; do
  keep=1
  for n in $ns; do [ "$o" == "build/inst_n$(printf %02d $n).o" ] && keep=0; done
  [ $keep == 1 ] && objs="$objs $o"
done
pids=""
for n in $ns; do
  nn=$(printf %02d $n)
  $NV $flags -c inst_n$nn.cu -o build_var/$name/inst_n$nn.o & pids="$pids $!"
  objs="$objs build_var/$name/inst_n$nn.o"
done
for p in $pids; do wait $p; done
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -o ../lib_$name/libpht.so $objs -cudart static -L/usr/local/cuda/lib64 -lnvrtc -Xlinker -rpath -Xlinker /usr/local/cuda/lib64
echo "lib_$name built"
