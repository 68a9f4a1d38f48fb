for K in 0 4096 8192 16384; do IRGL_HUB_KMAX=$K python tools/knob_probe.py 22 sssp IRGL_L2_PERSIST=0,1 ; done > gpurun_out/ab1_22.txt 2>&1
for K in 0 4096 8192 16384; do IRGL_HUB_KMAX=$K python tools/knob_probe.py 24 sssp IRGL_L2_PERSIST=0,1 ; done > gpurun_out/ab1_24.txt 2>&1
python tools/knob_probe.py 22 bfs IRGL_L2_PERSIST=0,1 >> gpurun_out/ab1_22.txt 2>&1
python tools/knob_probe.py 24 bfs IRGL_L2_PERSIST=0,1 >> gpurun_out/ab1_24.txt 2>&1
