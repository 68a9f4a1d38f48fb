python tools/knob_probe.py 22 sssp IRGL_FUSED=0,1 > gpurun_out/ab3.txt 2>&1
python tools/knob_probe.py 22 bfs IRGL_FUSED=0,1 >> gpurun_out/ab3.txt 2>&1
python tools/knob_probe.py 24 sssp IRGL_FUSED=0,1 >> gpurun_out/ab3.txt 2>&1
timeout 600 python -m pytest tests -m gpu -x -q --timeout 60 -p no:cacheprovider > gpurun_out/ab3_tests.txt 2>&1
