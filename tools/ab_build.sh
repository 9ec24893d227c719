#!/bin/bash
# Build the current tree (plus optional -D flags) into exp/<name>.so for A/B
# timing runs (load with DD_LIB=exp/<name>.so). Development aid.
set -e
name=$1; shift
DD_NVCC_DEFS="$*" python -m paper_2508_04917_b200.build --force > /dev/null
mkdir -p exp; cp paper_2508_04917_b200/libdd.so exp/$name.so
grep -A4 "k_apply_ringILi3ELj65536ELj16384ELb0ELi0ELi0E" paper_2508_04917_b200/build/ptxas.log | grep -E "registers" | sed "s/^/$name: /"
