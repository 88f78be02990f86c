#!/bin/bash
# Experiment library that differs from the base build only in epoch_grid.cu:
#   scripts/grid_variant.sh <name> "<-DFOO=1 ...>"   -> paper_1911_07722_b200/libsyscd_b200_<name>.so
# (recompiles that one file with the extra defines and links it with the base objects)
set -e
cd "$(dirname "$0")/.."
python -c "from paper_1911_07722_b200.csrc.build import build; build()" >/dev/null
C=paper_1911_07722_b200/csrc
mkdir -p $C/_obj_var
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC,-O2 \
  --expt-relaxed-constexpr -Xptxas -v $2 -c $C/epoch_grid.cu -o $C/_obj_var/epoch_grid_$1.o 2> $C/_obj_var/epoch_grid_$1.log
OBJS=$(ls $C/_obj/*.o | grep -v epoch_grid.o)
nvcc -shared -gencode arch=compute_100a,code=sm_100a $OBJS $C/_obj_var/epoch_grid_$1.o -o paper_1911_07722_b200/libsyscd_b200_$1.so -lcudart
echo paper_1911_07722_b200/libsyscd_b200_$1.so
# the test suite's build() must accept the variant as up to date (same sources, no extra flags in its env)
cp paper_1911_07722_b200/libsyscd_b200.so.sha256 paper_1911_07722_b200/libsyscd_b200_$1.so.sha256
