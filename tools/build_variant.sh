#!/bin/bash
# Build libfastatlas.so with extra nvcc flags into tools/lib_<name>.so, for
# A/B runs through FASTATLAS_LIB (tools/envcmp.sh "FASTATLAS_LIB=tools/lib_x.so"):
#   bash tools/build_variant.sh coop6 -DCOOP_MIN_BLOCKS=6
name=$1; shift
src=$(cd "$(dirname "$0")/../paper_2502_17712_b200/csrc" && pwd)
out=/tmp/fa_var_$name
mkdir -p $out
for f in fa_api fa_raster fa_charts fa_bounds fa_pack fa_uv fa_baselines fa_mesh; do
  /usr/local/cuda/bin/nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -lineinfo -fmad=false \
    -Xcompiler -fPIC --expt-relaxed-constexpr "$@" -c $src/$f.cu -o $out/$f.o &
  pids="$pids $!"
done
for p in $pids; do wait $p || { echo "build_variant: compile failed" >&2; exit 1; }; done
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -o "$(dirname "$0")/lib_$name.so" $out/*.o -lcudart
echo "built tools/lib_$name.so"
