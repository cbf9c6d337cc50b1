import sys; sys.path.insert(0,'.')
import numpy as np
import paper_2510_02894_b200 as sc
from paper_2510_02894_b200 import _native, synth
_native.set_option("stage_times", 2)  # per-stage events for last_kernel_times
m = synth.synth_mask("sphere", (24,24,24), radius=8)
for g in (0, 1):
    _native.set_option("graphs", g)
    try:
        r = sc.calculate_coefficients(m, (1,1,1))
        print("graphs", g, "ok", r.vertex_count, r.max_3d_diameter)
        r = sc.calculate_coefficients(m, (1,1,1))
        print("graphs", g, "ok2", r.vertex_count, r.max_3d_diameter, _native.last_kernel_times())
    except Exception as e:
        print("graphs", g, "ERR", e)
