for L in default variants/libirgl_rt_bcast.so; do
  if [ $L = default ]; then unset IRGL_LIB; else export IRGL_LIB=paper_1607_05707_b200/$L; fi
  echo "== $L"
  python tools/knob_probe.py 22 sssp IRGL_FUSED=1
  python tools/knob_probe.py 22 bfs IRGL_FUSED=1
  python tools/knob_probe.py 24 sssp IRGL_FUSED=1
  python tools/grid_probe.py 4096
done > gpurun_out/ab_barrier.txt 2>&1
