#!/bin/bash
# Free-running config-3 slice ingest vs CTA count (scripts/sm_ingest.cu):
# slice = ceil(4 MB / G) rounded up to 16 B, as many stages as fit 220 KB (<= 8)
for G in 96 104 112 116 120 124 128 132 136 140 145 148; do
  sl=$(( ( (4000000 + G - 1) / G + 15 ) / 16 * 16 ))
  S=$(( 225000 / sl )); [ $S -gt 8 ] && S=8
  ./scripts/sm_ingest_bin $G $sl $S > gpurun_out/sweep_$G.txt
  echo "G=$G slice=$sl S=$S $(sed -n 3p gpurun_out/sweep_$G.txt)"
done
