"""The device entropy (csrc/entropy.cuh) reproduces numpy's float64 sum order:
this pins that order -- pairwise summation with 8 accumulators per block of
<= 128 terms, split at n/2 rounded down to a multiple of 8 -- against np.sum
itself, in the same leaf/fold decomposition the kernel uses.  CPU only."""
import numpy as np
import pytest


def leaves(n):
    stack, out = [(0, n)], []
    while stack:
        b, m = stack.pop()
        if m <= 128:
            out.append((b, m))
        else:
            h = m // 2
            h -= h % 8
            stack.append((b + h, m - h))
            stack.append((b, h))
    return out


def leaf_sum(a, b, m):
    if m < 8:
        r = -0.0
        for i in range(m):
            r += a[b + i]
        return r
    acc = [a[b + j] for j in range(8)]
    i = 8
    while i < m - (m % 8):
        for j in range(8):
            acc[j] += a[b + i + j]
        i += 8
    res = ((acc[0] + acc[1]) + (acc[2] + acc[3])) + ((acc[4] + acc[5]) + (acc[6] + acc[7]))
    while i < m:
        res += a[b + i]
        i += 1
    return res


def fold(n, sums):
    stack, leaf, ret = [[n, 0, 0.0]], 0, 0.0
    while stack:
        top = stack[-1]
        m = top[0]
        if m <= 128:
            ret = sums[leaf]
            leaf += 1
            stack.pop()
            continue
        h = m // 2
        h -= h % 8
        if top[1] == 0:
            top[1] = 1
            stack.append([h, 0, 0.0])
        elif top[1] == 1:
            top[2], top[1] = ret, 2
            stack.append([m - h, 0, 0.0])
        else:
            ret = top[2] + ret
            stack.pop()
    return ret


@pytest.mark.parametrize("n", list(range(1, 140)) + [255, 256, 1000, 4097, 8192, 8193, 30001, 65536])
def test_leaf_fold_equals_numpy_sum(n):
    rng = np.random.default_rng(n)
    c = rng.integers(1, 9000, n)
    p = c / float(c.sum() + 7)
    t = p * np.log2(p)
    parts = leaves(n)
    assert all(m >= 64 for _, m in parts) or n <= 128
    assert len(parts) <= 1024
    got = fold(n, [leaf_sum(t, b, m) for b, m in parts])
    assert got == t.sum()
