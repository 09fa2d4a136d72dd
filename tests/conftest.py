import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
for p in (ROOT, os.path.join(ROOT, "oracle")):
    if p not in sys.path:
        sys.path.insert(0, p)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")


@pytest.fixture(scope="session")
def oracle():
    import oracle as o  # tests are the only importers of the oracle
    return o


def rnd_stream(seed):
    """Reference test RNG: mix64 chain -> uniform [-1, 1) (test_attention.cpp:13-24)."""
    import numpy as np
    import oracle as o
    state = [seed]

    def vec(n):
        out = np.empty(n, dtype=np.float32)
        for i in range(n):
            state[0] = o.mix64(state[0])
            out[i] = 2.0 * np.float32((state[0] >> 40) * 2.0**-24) - 1.0
        return out
    return vec


def upload_oracle_weights(W, mode="exact", device=0):
    """Upload an oracle WeightSet through the product C-ABI (tests only)."""
    import paper_2403_11421_b200 as sd
    tensors = [W.raw("embedding")]
    for l in range(W.spec.num_layers):
        for n in ("w_q", "w_k", "w_v", "w_o", "w_mlp_in", "w_mlp_out"):
            tensors.append(W.raw(n, l))
    tensors.append(W.raw("head"))
    s = W.spec
    spec = sd.make_model_spec(s.num_layers, s.model_dim, s.num_heads, s.mlp_dim, s.vocab_size,
                              s.num_kv_heads)
    return sd.DeviceWeights(spec, tensors, mode, device)
