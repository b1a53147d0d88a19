#!/usr/bin/env bash
# Build an A/B variant of libcurvalign_cuda.so with extra -D flags on the fused
# C1 translation unit (the other objects are the regular build/ ones):
#   tools/variant.sh NAME "-DCVA_FOO=1 -DCVA_BAR=2" [UNITS]   (UNITS: .cu names to
#   recompile with the flags, default "fused")
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
rm -f "$out/ptxas.log"
NVCC=${NVCC:-/usr/local/cuda/bin/nvcc}
ARCH="-gencode arch=compute_100a,code=sm_100a"
units=${3:-fused}
mine=""
skip="^$"
for u in $units; do
  src=paper_2501_17779_b200/csrc/$u.cu
  xcu=""
  if [ "$u" = capi ]; then src=paper_2501_17779_b200/csrc/capi.cpp; xcu="-x cu"; fi
  $NVCC $ARCH $flags -O3 -lineinfo -std=c++17 -Xcompiler -fPIC --expt-relaxed-constexpr -Xptxas -v \
    $xcu -c $src -o "$out/$u.o" 2>> "$out/ptxas.log"
  mine="$mine $out/$u.o"
  skip="$skip|/$u.o$"
done
objs=$(ls build/*.o | grep -Ev "$skip")
$NVCC $ARCH -shared -cudart static -o "$out/libcurvalign_cuda.so" $mine $objs
grep -A2 "v3.*resample_align_kernelILi1024" "$out/ptxas.log" | grep -E "registers|spill" || true
echo "built $out/libcurvalign_cuda.so"
