"""CC on the cut 4096^2 grid and TC on the triangulated grid, twice each (second = warm), for an
ncu launch list: python tools/profile_cctc.py"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1607_05707_b200 as irgl
ctx = irgl.Context()
g = ctx.generate_grid(4096, 4096, cut_period=512)
for _ in range(2):
    lab, st = irgl.cc(ctx, g)
print("CC", st.rounds, st.device_ms)
g.close()
g = ctx.generate_grid(4096, 4096, diag=True)
for _ in range(2):
    c, st = irgl.triangle_count(ctx, g)
print("TC", c, st.device_ms)
