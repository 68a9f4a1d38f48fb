#!/bin/bash
# ncu evidence for the bench's kernels (run under gpurun from the repo root):
#   one `ncu --set full` capture of the outlined kernel per workload (one warm traversal,
#   degree-ordered ids), summarised into gpurun_out/$TAG/ncu_<op>_rmat<scale>.json stamped with the
#   kernel-source hash (bench.py reads the DRAM traffic from the committed copy under profiles/),
#   and the launch list of the default bench command.
set -u
TAG=${1:-r2}
OUT=gpurun_out/$TAG
mkdir -p $OUT
for W in "sssp 22" "bfs 22" "sssp 24" "bfs 24"; do
  set -- $W
  timeout 900 ncu --set full --import-source on --clock-control none -k regex:persistent --launch-skip 1 -c 1 \
    -o $OUT/ncu_$1$2 -f python tools/one_traversal.py $1 $2 1 > $OUT/ncu_$1$2.log 2>&1
  NCU_KERNEL_REGEX=persistent python tools/ncu_json.py $OUT/ncu_$1$2.ncu-rep \
    "outlined persistent kernel, RMAT-$2 degree-ordered ids, one warm traversal (tools/one_traversal.py $1 $2 1)" \
    > $OUT/ncu_$1_rmat$2.json 2> $OUT/ncu_$1_rmat$2.err
  python tools/ncu_stalls.py $OUT/ncu_$1$2.ncu-rep 30 > $OUT/stalls_$1$2.txt 2>&1
  # the report itself stays on the box unless asked for (gpurun copies back <= 64 MiB)
  [ "${KEEP_NCU_REP:-0}" = 1 ] || rm -f $OUT/ncu_$1$2.ncu-rep
done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv \
  --log-file $OUT/launches_bench.csv python bench.py --steps 4 --warmup 3 --no-cpu-baseline --secondary 0 > $OUT/bench_under_ncu.log 2>&1
echo done
