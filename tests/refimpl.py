"""Independent plain-Python/numpy oracles used only by tests.

Restates the reference's test oracles (proj/tests/oracles.hpp:19-134) and its
RNG (rng.hpp:10-62) without sharing any code with either the C oracle or the
CUDA product, mirroring the reference's rule that test oracles share no code
path with the library under test (oracles.hpp:1-3).
"""
import math

import numpy as np

MASK = (1 << 64) - 1


def splitmix64(state):
    """Returns (output, new_state); rng.hpp:10-15."""
    state = (state + 0x9E3779B97F4A7C15) & MASK
    z = state
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & MASK
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & MASK
    return z ^ (z >> 31), state


def substream_seed(master, tag):
    a, s = splitmix64(master)
    s = a ^ ((tag * 0xD1B54A32D192ED03 + 0x8BB84B93962EACC9) & MASK)
    return splitmix64(s)[0]


def mix_tag(a, b, c=0, d=0):
    s = (a * 0x9E3779B97F4A7C15 + 1) & MASK
    for v in (b, c, d):
        out, s = splitmix64(s)  # right operand first: s is already advanced
        s ^= (out + v) & MASK
    return splitmix64(s)[0]


class PyRng:
    def __init__(self, seed):
        self.s = []
        sm = seed
        for _ in range(4):
            out, sm = splitmix64(sm)
            self.s.append(out)

    @staticmethod
    def _rotl(x, k):
        return ((x << k) | (x >> (64 - k))) & MASK

    def next_u64(self):
        s = self.s
        result = (self._rotl((s[0] + s[3]) & MASK, 23) + s[0]) & MASK
        t = (s[1] << 17) & MASK
        s[2] ^= s[0]
        s[3] ^= s[1]
        s[1] ^= s[2]
        s[0] ^= s[3]
        s[2] ^= t
        s[3] = self._rotl(s[3], 45)
        return result

    def uniform(self):
        return (self.next_u64() >> 11) * 2.0 ** -53

    def below(self, bound):
        return (self.next_u64() * bound) >> 64

    def gaussian(self):
        u1 = 1.0 - self.uniform()
        u2 = self.uniform()
        return math.sqrt(-2.0 * math.log(u1)) * math.cos(2.0 * math.pi * u2)


def pinv_solve(a, y):
    """One-sided Jacobi pseudo-inverse solve (oracles.hpp:19-72)."""
    b = np.array(a, dtype=np.float64).T.copy()  # columns as rows
    m = b.shape[0]
    v = np.eye(m)
    tol = 1e-15
    for _ in range(60):
        rotated = False
        for p in range(m - 1):
            for q in range(p + 1, m):
                app = b[p] @ b[p]
                aqq = b[q] @ b[q]
                apq = b[p] @ b[q]
                if abs(apq) <= tol * math.sqrt(app * aqq):
                    continue
                rotated = True
                zeta = (aqq - app) / (2.0 * apq)
                t = (1.0 if zeta >= 0 else -1.0) / (abs(zeta) + math.sqrt(1.0 + zeta * zeta))
                cs = 1.0 / math.sqrt(1.0 + t * t)
                sn = cs * t
                bp = b[p].copy()
                b[p] = cs * bp - sn * b[q]
                b[q] = sn * bp + cs * b[q]
                vp = v[p].copy()
                v[p] = cs * vp - sn * v[q]
                v[q] = sn * vp + cs * v[q]
        if not rotated:
            break
    w = np.zeros(m)
    for j in range(m):
        sigma = math.sqrt(b[j] @ b[j])
        if sigma <= 0:
            continue
        uty = (b[j] / sigma) @ y
        w += v[j] * uty / sigma
    return w


def reference_forward(dims, w0, layers, final, x):
    """Straight-line evaluation (oracles.hpp:75-96); layers = [(W, b)]."""
    x = np.asarray(x, dtype=np.float64)
    lin = x @ w0
    act = x
    for W, b in layers:
        act = np.maximum(act @ W.T + b, 0.0)
    return lin + act @ final


class ReferenceAdam:
    """Flat-vector Adam (oracles.hpp:99-115)."""

    def __init__(self, size, lr):
        self.m = np.zeros(size)
        self.v = np.zeros(size)
        self.t = 0
        self.lr, self.beta1, self.beta2, self.eps = lr, 0.9, 0.999, 1e-8

    def step(self, theta, grad):
        self.t += 1
        self.m = self.beta1 * self.m + (1 - self.beta1) * grad
        self.v = self.beta2 * self.v + (1 - self.beta2) * grad * grad
        mhat = self.m / (1 - self.beta1 ** self.t)
        vhat = self.v / (1 - self.beta2 ** self.t)
        theta -= self.lr * mhat / (np.sqrt(vhat) + self.eps)
