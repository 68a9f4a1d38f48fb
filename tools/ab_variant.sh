#!/bin/bash
# A/B of the in-tree library against one build variant (tools/build_variant.sh NAME FLAGS):
#   tools/ab_variant.sh NAME OUTFILE   (RMAT-22 / RMAT-24 SSSP and BFS, degree-ordered ids)
V=$1; OUT=$2
for L in default paper_1607_05707_b200/variants/libirgl_rt_$V.so; do
  if [ $L = default ]; then unset IRGL_LIB; else export IRGL_LIB=$L; fi
  echo "== $L"
  python tools/knob_probe.py 22 sssp IRGL_X=0
  python tools/knob_probe.py 22 bfs IRGL_X=0
  python tools/knob_probe.py 24 sssp IRGL_X=0
  python tools/knob_probe.py 24 bfs IRGL_X=0
done > $OUT 2>&1
