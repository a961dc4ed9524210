import sys, os
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2306_03078_b200 as P
from paper_2306_03078_b200 import synth
for (m, n, bw, rate, perm) in [(32, 256, 3, 0.0, False), (32, 256, 3, 0.02, False), (96, 544, 3, 0.02, True)]:
    a = synth.make_layer(m, n, weight_bits=bw, scale_bits=bw, zero_bits=bw, seed=m, permute=perm, outlier_rate=rate)
    s = P.encode_arrays(a)
    host = P.debug_tiled_host(s)
    dev = P.Layer(s).debug_cells()
    print(m, n, "off equal", np.array_equal(dev["cell_off"], host["cell_off"]), host["cell_off"][:4], dev["cell_off"][:4])
    hc, dc = host["cells"], dev["cells"]
    print("  sizes", hc.size, dc.size)
    d = np.nonzero(hc[: dc.size] != dc)[0]
    print("  ndiff", d.size, "first", d[:10], "unit bytes", host["cell_bytes"] // 2)
    if d.size:
        i = d[0]
        print("  host", hc[i:i + 16], "\n  dev ", dc[i:i + 16])
