"""Model of K1's value-slot assignment (transform.cu step 6c) on CPU.

K1 assigns forward-pass value slots by a warp-parallel interval colouring:
value v (the distinct inputs first, then the ops in order) starts at time v
and ends at Ip + (its last reader's op index), right after it starts (an op
value nobody reads) or never (outputs, inputs nobody reads); the slot count is
the maximum overlap M; start s < M takes slot s, start s >= M the slot freed
by the (s - M)-th end event (time order, ties by value index), resolved by
pointer jumping.  This test restates that algorithm in numpy and checks, on
random op sequences, that it is a valid colouring (no two live values share a
slot -- K2 reads every value from its slot while it is live) and that it uses
exactly as many slots as the lowest-free-slot scan it replaced (both optimal).
"""
import numpy as np
import pytest

INF = 1 << 30


def intervals(rng, n_in, n_ops):
    """(start, end) per value for a random DAG: op k reads earlier values."""
    V = n_in + n_ops
    last = np.full(V, -1)                      # last reader's op index
    for k in range(n_ops):
        srcs = rng.choice(n_in + k, size=min(n_in + k, rng.integers(1, 6)), replace=False)
        last[srcs] = k
    outputs = rng.choice(np.arange(n_in, V), size=min(n_ops, 2), replace=False) if n_ops else []
    ends = []
    for v in range(V):
        if v in outputs:
            e = INF
        elif last[v] < 0:
            e = INF if v < n_in else v + 1
        else:
            e = n_in + last[v]
        ends.append(e)
    return np.arange(V), np.array(ends)


def fifo_colouring(starts, ends):
    V = len(starts)
    live = [(t + 1) - sum(1 for e in ends if e <= t) for t in range(V)]
    M = max(live) if V else 0
    order = sorted((e, v) for v, e in enumerate(ends) if e != INF)
    src = [v for _, v in order]
    par = [v if v < M else src[v - M] for v in range(V)]
    while True:  # pointer jumping
        nxt = [par[par[v]] for v in range(V)]
        if nxt == par:
            break
        par = nxt
    return M, par


def greedy_colouring(starts, ends):
    slots, used = [0] * len(starts), set()
    free_at = {}
    n = 0
    for v in range(len(starts)):
        for sl in free_at.pop(v, []):
            used.discard(sl)
        sl = min(set(range(len(starts) + 1)) - used)
        used.add(sl)
        slots[v] = sl
        n = max(n, sl + 1)
        if ends[v] != INF:
            free_at.setdefault(ends[v], []).append(sl)
    return n, slots


@pytest.mark.parametrize("seed", range(40))
def test_fifo_colouring_valid_and_optimal(seed):
    rng = np.random.default_rng(seed)
    n_in, n_ops = int(rng.integers(1, 8)), int(rng.integers(0, 60))
    starts, ends = intervals(rng, n_in, n_ops)
    M, slot = fifo_colouring(starts, ends)
    n_greedy, _ = greedy_colouring(starts, ends)
    assert M == n_greedy
    assert all(0 <= s < max(M, 1) for s in slot)
    for a in range(len(starts)):
        for b in range(a + 1, len(starts)):
            overlap = starts[a] < ends[b] and starts[b] < ends[a]
            assert not (overlap and slot[a] == slot[b]), (a, b)
