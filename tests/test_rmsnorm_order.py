"""CPU pin for the RMSNorm -> INT producer's summation order (serq_rmsnorm_quant_int).

The kernel reproduces the reference's float64 row mean of squares (saliency.py:194-196 via
np.mean) bit for bit by replaying NumPy's pairwise summation: leaves of <= 128 elements summed
with eight strided accumulators combined ((r0+r1)+(r2+r3))+((r4+r5)+(r6+r7)) plus the in-order
tail, leaves joined along the recursion that splits n at n/2 rounded down to a multiple of 8.
This test restates that order in Python (the same tree the C host code builds) and checks it
against np.mean on rows chosen so that any other association order would round differently.
"""

import numpy as np
import pytest


def _leaf(a):
    n = a.size
    if n < 8:
        s = 0.0
        for v in a:
            s += v
        return s
    r = [a[j] for j in range(8)]
    body = n - n % 8
    for i in range(8, body, 8):
        for j in range(8):
            r[j] += a[i + j]
    s = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]))
    for i in range(body, n):
        s += a[i]
    return s


def _pairwise(a):
    n = a.size
    if n <= 128:
        return _leaf(a)
    n2 = n // 2
    n2 -= n2 % 8
    return _pairwise(a[:n2]) + _pairwise(a[n2:])


@pytest.mark.parametrize("K", [1, 7, 8, 100, 128, 129, 1000, 2560, 3008, 4096, 4100, 8192])
def test_pairwise_replay_matches_numpy_mean(K):
    rng = np.random.default_rng(K)
    # heavy-tailed magnitudes spanning ~2^40 make the f64 sum order-sensitive
    x = rng.standard_normal((6, K)) * np.exp2(rng.uniform(-20, 20, (6, K)))
    sq = x * x
    ref = np.mean(sq, axis=1)
    for i in range(x.shape[0]):
        assert _pairwise(sq[i]) / K == ref[i]


def test_sequential_order_would_differ():
    # the replay is not vacuous: a plain left-to-right sum rounds differently on these rows
    rng = np.random.default_rng(0)
    x = rng.standard_normal((6, 4096)) * np.exp2(rng.uniform(-20, 20, (6, 4096)))
    sq = x * x
    seq = np.array([sum(float(v) for v in row) for row in sq]) / 4096
    assert (seq != np.mean(sq, axis=1)).any()
