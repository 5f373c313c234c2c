"""Seeded fixture builders restating the reference tests' helpers.

random_mat / random_design: test_lls.cpp:13-19, test_hybrid_nn.cpp:23-29.
make_w0: test_hybrid_nn.cpp:15-21.
random_net: test_hybrid_nn.cpp:33-41 (final scale 0.5) and test_fused.cpp:29-40
(w0 drawn from the same stream first, final scale 0.3).
"""
import numpy as np

from oracle import oracle as O


def random_mat(rows, cols, seed):
    r = O.Rng(seed)
    return np.array([[r.gaussian() for _ in range(cols)] for _ in range(rows)], dtype=np.float64)


def make_w0(width, seed):
    r = O.Rng(seed)
    return np.array([r.gaussian() for _ in range(width)])


def random_net_hybrid(dims, seed):
    rng = O.Rng(seed)
    net = O.init_params(dims, make_w0(dims[0], seed + 1), rng)
    layers, final = net.layers()
    for _, b in layers:
        for i in range(b.size):
            b[i] = rng.gaussian() * 0.1
    for i in range(final.size):
        final[i] = rng.gaussian() * 0.5
    return net


def random_net_fused(dims, seed):
    rng = O.Rng(seed)
    w0 = np.array([rng.gaussian() for _ in range(dims[0])])
    net = O.init_params(dims, w0, rng)
    layers, final = net.layers()
    for _, b in layers:
        for i in range(b.size):
            b[i] = rng.gaussian() * 0.1
    for i in range(final.size):
        final[i] = rng.gaussian() * 0.3
    return net


def max_rel_dev(a, b):
    scale = max(1e-30, float(np.max(np.abs(b))))
    return float(np.max(np.abs(np.asarray(a) - np.asarray(b)))) / scale


def seq_matvec(x, w):
    """x @ w with the contraction summed left to right (the oracle's order)."""
    x = np.asarray(x, dtype=np.float64)
    acc = np.zeros(x.shape[0])
    for c in range(x.shape[1]):
        acc = acc + x[:, c] * w[c]
    return acc


def record(name, **vals):
    """Append measured parity numbers to $NOMA_PARITY_LOG (JSON lines)."""
    import json
    import os

    path = os.environ.get("NOMA_PARITY_LOG")
    if not path:
        return
    with open(path, "a") as f:
        f.write(json.dumps({"test": name, **{k: (float(v) if not isinstance(v, (str, list)) else v)
                                               for k, v in vals.items()}}) + "\n")
