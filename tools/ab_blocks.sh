# block size x per-warp staging size variants (tools/build_variant.sh), SSSP / BFS RMAT-22 / 24
for V in "$@"; do bash tools/ab_variant.sh $V gpurun_out/ab_$V.txt; done
