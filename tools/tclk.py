"""Developer probe: per-CTA phase timeline of the tree group kernels (library built with -DMABD_EXP_TCLOCK).
    MABD_LIB=build_variants/lib_tclk.so python tools/tclk.py [depth]
Slots per CTA: 0 start, 1 stages 1-2 + leaves done, 2.. up levels (deepest first), 32 down start, 33.. down levels
(shallowest first... indexed by level offset), 63 end. Prints, per mode, the median / max over CTAs of each phase."""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from mabd_scenes import generators as G  # noqa: E402
from paper_2603_08079_b200 import Simulator  # noqa: E402

d = int(sys.argv[1]) if len(sys.argv) > 1 else 16
sc = G.cfg4_binary_tree(d)
sim = Simulator.from_scene(sc)
sim.prefactor(sc.h)
sim.step(sc.h, 3)
torch.cuda.synchronize()
lib = sim._lib
n = 3 * 512 * 64
buf = (ctypes.c_ulonglong * n)()
lib.mabd_dbg_tclk.argtypes = [ctypes.c_void_p, ctypes.c_int]
assert lib.mabd_dbg_tclk(ctypes.addressof(buf), n) == 0
T = np.frombuffer(buf, dtype=np.uint64).astype(np.int64).reshape(3, 512, 64)
for mode, name in ((0, "UP"), (2, "TOP (both)"), (1, "DOWN")):
    t = T[mode]
    ctas = np.where(t.max(axis=1) > 0)[0]
    t = t[ctas]
    slots = [s for s in range(64) if (t[:, s] > 0).all()]
    slots.sort(key=lambda s: np.median(t[:, s]))  # in time order
    print(f"== {name}: {len(ctas)} CTAs; kernel span (first mark → last mark) {((t[:, slots].max() - t[:, slots][:, 0].min()) / 1e3):.1f} us")
    prev = None
    for s in slots:
        if prev is not None:
            dt = (t[:, s] - t[:, prev]) / 1e3
            print(f"  slot {prev:2d}->{s:2d}: median {np.median(dt):7.2f} us  max {dt.max():7.2f} us")
        prev = s
e = T[0, 0, 40:45]
print("elim probe (last body of CTA 0, last kernel to write):", [round((int(e[i + 1]) - int(e[i])) / 1e3, 2) for i in range(4)],
      "us: column load | children | Gauss-Jordan | outputs")
e = T[0, 0, 50:53]
print("lambda probe (root of group 0, DOWN):", [round((int(e[i + 1]) - int(e[i])) / 1e3, 2) for i in range(2)],
      "us: λ_u load | y − Wλ_u")
e = T[0, 0, 55:59]
print("update probe (thread 0 of CTA 0, DOWN0):", [round((int(e[i + 1]) - int(e[i])) / 1e3, 2) for i in range(3)],
      "us: R/H/λ_u loads | child points (λ, ȳ) | H⁻¹ apply + stores")
