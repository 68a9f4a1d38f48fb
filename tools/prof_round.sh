#!/bin/bash
# One GPU call's worth of evidence for the dominant kernel (run under gpurun from the repo root):
#   round trace of one SSSP RMAT-22 traversal (degree-ordered ids), the ncu launch list of the
#   bench command, and one `ncu --set full` capture of the outlined SSSP kernel with source.
# usage: tools/prof_round.sh TAG [op] [scale]
set -u
TAG=${1:-r2}; OP=${2:-sssp}; SCALE=${3:-22}
OUT=gpurun_out/$TAG
mkdir -p $OUT
RELABEL=1 timeout 300 python tools/round_trace.py $SCALE $OP > $OUT/round_trace_${OP}${SCALE}.txt 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file $OUT/launches_${OP}${SCALE}.csv python bench.py --op $OP --scale $SCALE --steps 4 --warmup 3 --no-cpu-baseline > $OUT/bench_under_ncu.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:persistent --launch-skip 1 -c 1 \
  -o $OUT/ncu_${OP}${SCALE} -f python tools/one_traversal.py $OP $SCALE 1 > $OUT/ncu_${OP}${SCALE}.log 2>&1
echo done
