"""Dump K1 net blocks for a fixed set of populations (valid and corrupt) so two
builds of the library can be compared byte for byte (run once per build, then
`python scripts/k1_dump.py cmp a.npz b.npz`).  Test infrastructure."""
import ctypes as C
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))


def cases():
    import oracle_lib as ol
    from paper_2504_08339_b200 import synthetic
    from test_oracle_vs_ref import _corrupt
    out = []
    for (P, N, Cc, fill, na, ng, seed) in [(2000, 64, 256, 0.75, 1, 1, 0), (1000, 64, 256, 1.0, 5, 4, 1),
                                            (300, 128, 1024, 0.75, 1, 1, 2), (300, 16, 32, 1.0, 5, 4, 3),
                                            (200, 255, 1024, 0.9, 5, 4, 4)]:
        n, c = synthetic.synthetic_population(P, N, Cc, fill=fill, n_act=na, n_agg=ng, seed=seed)
        rng = np.random.default_rng(100 + seed)
        for i in range(0, P, 2):  # shuffled node and connection rows in every other genome
            n[i] = n[i][rng.permutation(N)]
            c[i] = c[i][rng.permutation(Cc)]
        out.append((f"syn{N}_{Cc}_{fill}", N, Cc, None, n, c, na, ng))
    # keys past 2^23 (the transform's wide-key rank path): hidden keys shifted up
    n, c = synthetic.synthetic_population(500, 64, 256, fill=0.75, seed=9)
    for a in (n[..., 0], c[..., 0], c[..., 1]):
        a[a >= 5] += 20_000_000
    out.append(("bigkeys", 64, 256, None, n, c, 1, 1))
    for seed, (N, Cc) in [(71, (16, 60)), (90210, (50, 100)), (1312, (40, 200))]:
        n, c = ol.random_genomes(seed, ol.RICH, 300, N, Cc)
        rng = np.random.default_rng(seed)
        kinds = [None, "cycle", "selfloop", "dangling", "bad_act", "bad_agg", "missing_output", "dup_pair"]
        for i in range(n.shape[0]):
            k = kinds[i % len(kinds)]
            if k:
                n[i], c[i] = _corrupt(n[i], c[i], rng, k)
        out.append((f"rand{seed}", N, Cc, "ref", n, c, 5, 4))
    return out


def dump(path):
    import torch
    import oracle_lib as ol
    import paper_2504_08339_b200 as m
    res = {}
    for name, N, Cc, keys, n, c, na, ng in cases():
        if keys == "ref":
            ik, ok = [0, 1, 2], [3]
            schema = m.AttributeSchema(list(ol.RICH.activations), list(ol.RICH.aggregations))
        else:
            ik, ok = [0, 1, 2, 3], [4]
            acts = ["tanh", "sigmoid", "identity", "relu", "sin"][:na]
            aggs = ["sum", "product", "max", "mean"][:ng]
            schema = m.AttributeSchema(acts, aggs)
        eng = m.Engine(m.GenomeLimits(N, Cc), ik, ok, schema)
        dn = torch.from_numpy(np.ascontiguousarray(n)).cuda()
        dc = torch.from_numpy(np.ascontiguousarray(c)).cuda()
        nets = torch.zeros(n.shape[0] * eng.net_bytes, dtype=torch.uint8, device="cuda")
        st = eng._lib.fnb_transform_d(eng._h, dn.data_ptr(), dc.data_ptr(), n.shape[0], nets.data_ptr(), None)
        torch.cuda.synchronize()
        res[name] = nets.cpu().numpy().reshape(n.shape[0], eng.net_bytes)
        print(name, "status", st, file=sys.stderr)
    np.savez(path, **res)


def cmp(a, b):
    A, B = np.load(a), np.load(b)
    bad = 0
    for k in A.files:
        x, y = A[k], B[k]
        d = np.where((x != y).any(axis=1))[0]
        st = x[:, :4].copy().view(np.int32)[:, 0]
        print(k, "genomes", x.shape[0], "failing", int((st != 0).sum()), "differ", len(d),
              "(failing among them:", int((st[d] != 0).sum()), ")")
        if len(d):
            i = d[0]
            j = np.where(x[i] != y[i])[0]
            print("   first genome", i, "status", st[i], "bytes", j[:16])
        bad += len(d)
    print("TOTAL_DIFF", bad)


if __name__ == "__main__":
    if sys.argv[1] == "cmp":
        cmp(sys.argv[2], sys.argv[3])
    else:
        dump(sys.argv[1])
