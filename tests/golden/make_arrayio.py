"""Generate ArrayFile fixtures with the reference's own writer (run in the
build container, where /root/reference is importable).  The committed files
pin this package's reader/writer to the reference format byte for byte;
arrayio_ref.npz holds the arrays that were written."""
import os
import sys

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")
from hicu.arrayio import write_array  # noqa: E402

out = os.path.dirname(os.path.abspath(__file__))
rng = np.random.default_rng(7)
arrays = {
    "c16": rng.standard_normal((3, 4, 2)) + 1j * rng.standard_normal((3, 4, 2)),
    "f8": rng.standard_normal((5,)),
    "u1": (rng.random((2, 3, 4)) < 0.5).astype(np.uint8),
}
for k, a in arrays.items():
    write_array(os.path.join(out, f"arrayio_{k}.hicu"), a)
np.savez(os.path.join(out, "arrayio_ref.npz"), **arrays)
