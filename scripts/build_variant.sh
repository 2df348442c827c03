#!/bin/bash
# Build a library variant for A/B runs: scripts/build_variant.sh NAME [nvcc -D flags...]
# -> exp_libs/NAME.so (scripts/gpu_ab_libs.sh runs every exp_libs/*.so in turn).
set -e
cd "$(dirname "$0")/.."
name=$1; shift
mkdir -p exp_libs build/var_$name build/obj
make lib > /dev/null   # host objects
for f in decoder harness; do
  /usr/local/cuda/bin/nvcc -O3 -std=c++20 -gencode arch=compute_100a,code=sm_100a -lineinfo -Xcompiler -fPIC,-Wall \
    -Ipaper_2507_03509_b200/csrc -Iinclude "$@" -c paper_2507_03509_b200/csrc/$f.cu -o build/var_$name/$f.o &
done
wait
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -cudart static -o exp_libs/$name.so \
  build/obj/code.o build/obj/c_api.o build/obj/devmem.o build/var_$name/decoder.o build/var_$name/harness.o -lpthread
echo "built exp_libs/$name.so"
