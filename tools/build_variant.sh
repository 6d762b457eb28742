#!/bin/bash
# A/B builds of compile-time variants: tools/build_variant.sh NAME "-DKNOB=V ..."
# -> variants/libnpsd_b200_NAME.so (select with NPSD_B200_LIB=...; git-ignored,
# travels to the GPU box with gpurun)
set -e
cd "$(dirname "$0")/.."
mkdir -p variants/obj_$1
NVCC=/usr/local/cuda/bin/nvcc
ARCH="-gencode arch=compute_100a,code=sm_100a"
$NVCC $ARCH -O3 -lineinfo -std=c++17 --fmad=false -Xcompiler -fPIC,-ffp-contract=off -ccbin /usr/bin/g++ $2 \
    -c paper_2310_00177_b200/csrc/npsd_b200.cu -o variants/obj_$1/npsd_b200.o
$NVCC $ARCH -shared -ccbin /usr/bin/g++ -o variants/libnpsd_b200_$1.so variants/obj_$1/npsd_b200.o \
    paper_2310_00177_b200/csrc/host.o -lcudart_static -lrt -lpthread -ldl
echo built variants/libnpsd_b200_$1.so
