"""Golden fixtures of the reference's dense Cadzow baseline
(``hicu.oracle.cadzow_complete``, pkg/src/hicu/oracle.py:144-174): the
reference run on the small recovery problem of make_golden.py (24x24x3,
5x5x3 kernel, rank 49, 1 % noise), non-circular and circular, 12 sweeps.

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden_cadzow.py
"""

import os
import sys

import numpy as np

REF = os.environ.get("HICU_REFERENCE_SRC", "/root/reference/pkg/src")
sys.path.insert(0, REF)
HERE = os.path.dirname(os.path.abspath(__file__))

from hicu import KernelMask  # noqa: E402
from hicu.oracle import cadzow_complete  # noqa: E402

g = dict(np.load(os.path.join(HERE, "golden_recon.npz"), allow_pickle=False))
x0, mask, ref = g["lp_x0"], g["lp_mask"], g["lp_ref"]
kern = KernelMask.full(tuple(int(v) for v in g["lp_kext"]))
out = {}
for name, circ in (("cadzow", ()), ("cadzow_circ", (0, 1))):
    trace = []
    x = cadzow_complete(x0, mask, kern, 49, 12, circular_axes=circ,
                        callback=lambda it, xx: trace.append(float(np.linalg.norm(xx))))
    out[name + "_x"] = x
    out[name + "_norms"] = np.array(trace)
np.savez_compressed(os.path.join(HERE, "golden_cadzow.npz"), **out)
print("wrote golden_cadzow.npz")
