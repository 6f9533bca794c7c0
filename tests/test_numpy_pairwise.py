"""CPU pin of numpy's pairwise summation, the order ssk_pairwise_sum reproduces on the device.

np.add.reduce over a contiguous float64 array: 0.0 + pairwise(all n), where a node of n
elements is summed sequentially (n < 8), with eight interleaved accumulators combined as
((r0+r1)+(r2+r3))+((r4+r5)+(r6+r7)) plus a sequential tail (n <= 128), else split at
n2 = n//2 - (n//2) % 8 into left + right (numpy/_core/src/umath/loops_utils.h.src).
The kernel's two-level evaluation (complete top tree of depth d, subtree sums, level-by-
level combination) is restated here too and must give the same bits.
"""

import numpy as np
import pytest


def pairwise(a, off, n):
    if n < 8:
        r = 0.0
        for i in range(n):
            r += a[off + i]
        return r
    if n <= 128:
        r = [a[off + j] for j in range(8)]
        i = 8
        while i < n - n % 8:
            for j in range(8):
                r[j] += a[off + i + j]
            i += 8
        res = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]))
        while i < n:
            res += a[off + i]
            i += 1
        return res
    n2 = n // 2
    n2 -= n2 % 8
    return pairwise(a, off, n2) + pairwise(a, off + n2, n - n2)


def two_level(a):
    """The kernel's evaluation (pool_exact.cu): depth d top tree, subtrees, combination."""
    n = len(a)
    d = 0
    while d < 15 and (n >> (d + 1)) > 256:
        d += 1
    leaves = []
    for t in range(1 << d):
        off, ln = 0, n
        for lv in range(d - 1, -1, -1):
            n2 = ln // 2
            n2 -= n2 % 8
            if (t >> lv) & 1:
                off, ln = off + n2, ln - n2
            else:
                ln = n2
        leaves.append(pairwise(a, off, ln))
    while len(leaves) > 1:
        leaves = [leaves[2 * j] + leaves[2 * j + 1] for j in range(len(leaves) // 2)]
    return 0.0 + leaves[0]


@pytest.mark.parametrize("n", list(range(1, 140)) + [255, 256, 257, 1000, 4099, 65536, 100003, 252004])
def test_emulation_matches_numpy(n):
    a = np.random.default_rng(n).uniform(-1.0, 1.0, n) * 10.0 ** np.random.default_rng(n + 1).integers(-3, 4, n)
    want = np.add.reduce(a)
    lst = a.tolist()
    assert 0.0 + pairwise(lst, 0, n) == want
    if n >= 1000:
        assert two_level(lst) == want
    assert np.mean(a) == want / n
