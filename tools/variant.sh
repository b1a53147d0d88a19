#!/bin/bash
# Build libcurvalign_cuda.so with extra -D flags into build/var_<name>.so (experiments):
#   tools/variant.sh name -DFOO=1 ...   then   CVA_LIB_PATH=build/var_name.so python tools/bench_parts.py
set -e
name=$1; shift
cd "$(dirname "$0")/.."
mkdir -p build/var_$name
ARCH="-gencode arch=compute_100a,code=sm_100a"
FL="$ARCH -O3 -lineinfo -std=c++17 -Xcompiler -fPIC --expt-relaxed-constexpr $*"
objs=""
for f in kernels fused allpairs largen elastic dropin_kernels gfft probe; do
  /usr/local/cuda/bin/nvcc $FL -c paper_2501_17779_b200/csrc/$f.cu -o build/var_$name/$f.o &
  objs="$objs build/var_$name/$f.o"
done
/usr/local/cuda/bin/nvcc $FL -x cu -c paper_2501_17779_b200/csrc/capi.cpp -o build/var_$name/capi.o &
wait
/usr/local/cuda/bin/nvcc $ARCH -shared -cudart static -o build/var_$name.so $objs build/var_$name/capi.o
echo build/var_$name.so
