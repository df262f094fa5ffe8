"""Compare two dumped psi arrays: bitwise equality and relative L2 difference."""
import sys
import numpy as np
a, b = np.load(sys.argv[1]), np.load(sys.argv[2])
eq = np.array_equal(a.view(np.uint32), b.view(np.uint32))
d = np.linalg.norm((a - b).astype(np.float64)) / max(np.linalg.norm(b.astype(np.float64)), 1e-300)
nd = int(np.sum(np.any(a.view(np.uint32) != b.view(np.uint32), axis=-1)))
print(f"bitwise_equal={eq} rel_l2={d:.3e} differing_px={nd} of {a.shape[0] * a.shape[1]}")
