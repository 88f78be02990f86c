#!/bin/bash
# Build an experiment variant library: scripts/build_variant.sh <name> "<-DFOO=1 ...>"
SYSCD_LIB_NAME=libsyscd_b200_$1.so SYSCD_NVCC_DEFS="$2" python -c "from paper_1911_07722_b200.csrc.build import build; print(build())"
