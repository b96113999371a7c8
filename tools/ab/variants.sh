#!/bin/bash
# build experiment variants of the engine library into scratch/lib_<name>.so
set -e
mkdir -p "$(dirname "$0")/../../scratch"
cd "$(dirname "$0")/../.."
build() { name=$1; shift; nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -fmad=false -std=c++17 -Xcompiler -fPIC,-ffp-contract=off -shared "$@" -o scratch/lib_$name.so paper_2601_11546_b200/csrc/engine.cu paper_2601_11546_b200/csrc/trace_v1.cpp; }
for spec in "$@"; do name=${spec%%:*}; defs=${spec#*:}; build $name $defs & done; wait
