# E1 scheduler sweep (RMAT-22 BFS + SSSP defer 1024): bash tools/sched_sweep.sh "wt..." "ce..." "ct..."
for wt in ${1:-64 128}; do for ce in ${2:-256 512}; do for ct in ${3:-512}; do CTX="{\"warp_threshold\": $wt, \"chunk_edges\": $ce, \"cta_threshold\": $ct}" timeout 120 python tools/defer_sweep.py 22 1024; done; done; done
