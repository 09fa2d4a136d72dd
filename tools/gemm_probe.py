"""Minimal tcgen05 GEMM probe: one apply_linear in bf16 mode vs numpy."""
import os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2403_11421_b200 as sd
D = int(sys.argv[1]) if len(sys.argv) > 1 else 256
F, V = 512, 512
B = int(sys.argv[3]) if len(sys.argv) > 3 else 128
mode = sys.argv[2] if len(sys.argv) > 2 else "bf16"
spec = sd.make_model_spec(1, D, 2, F, V)
rng = np.random.default_rng(0)
t = [rng.uniform(-1, 1, D * V).astype(np.float32)]
shapes = [(D, D), (D, D), (D, D), (D, D), (F, D), (D, F)]
for (o, i) in shapes:
    t.append(rng.uniform(-1, 1, o * i).astype(np.float32))
t.append(rng.uniform(-1, 1, V * D).astype(np.float32))
w = sd.DeviceWeights(spec, t, mode)
x = rng.uniform(-1, 1, (B, D)).astype(np.float32)
y = sd.apply_linear(w, 0, 4, x)
wT = t[4].reshape(D, D)  # column-major (out x in) == row-major [in][out]
ref = x.astype(np.float64) @ wT.astype(np.float64)
print("max abs err", float(np.abs(y - ref).max()), "max |ref|", float(np.abs(ref).max()))
