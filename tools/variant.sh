#!/usr/bin/env bash
# Build an A/B variant of libcurvalign_cuda.so with extra -D flags on the fused
# C1 translation unit (the other objects are the regular build/ ones):
#   tools/variant.sh NAME "-DCVA_FOO=1 -DCVA_BAR=2"
# -> build/var_NAME/libcurvalign_cuda.so; select it at run time with
#   CVA_LIB_PATH=build/var_NAME/libcurvalign_cuda.so python tools/bench_parts.py
# Development only (never shipped; build/ travels to the GPU box with gpurun).
set -euo pipefail
cd "$(dirname "$0")/.."
name=$1
flags=${2:-}
make -s lib >/dev/null
out=build/var_$name
mkdir -p "$out"
NVCC=${NVCC:-/usr/local/cuda/bin/nvcc}
ARCH="-gencode arch=compute_100a,code=sm_100a"
$NVCC $ARCH $flags -O3 -lineinfo -std=c++17 -Xcompiler -fPIC --expt-relaxed-constexpr -Xptxas -v \
  -c paper_2501_17779_b200/csrc/fused.cu -o "$out/fused.o" 2> "$out/ptxas.log"
objs=$(ls build/*.o | grep -v '/fused.o$')
$NVCC $ARCH -shared -cudart static -o "$out/libcurvalign_cuda.so" "$out/fused.o" $objs
grep -A2 "v3.*resample_align_kernelILi1024" "$out/ptxas.log" | grep -E "registers|spill" || true
echo "built $out/libcurvalign_cuda.so"
