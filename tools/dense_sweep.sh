# dense-round threshold sweep (RMAT-22 BFS + SSSP defer 1024): bash tools/dense_sweep.sh "div..."
for dd in ${1:--1 8 16 32 64}; do CTX="{\"dense_div\": $dd}" timeout 120 python tools/defer_sweep.py ${2:-22} 1024; done
