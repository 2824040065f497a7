"""Pins for the CPU oracle (no GPU).  Each pin is independent of the oracle's own code:

* an independent python brute force over all 2^N labelings of the cut capacity of
  SURVEY.md §8(c) (the plain definition of F* and of the inclusion-minimal minimiser);
* scipy's maximum_flow (a library max-flow) on medium grids, with the canonical mask
  recomputed here from scipy's flow;
* SPEC worked examples (tests/golden/spec_examples.json, each cited);
* closed forms (no n-links; strong coupling);
* properties: duality cut(mask) == F, monotonicity, t-link normalisation invariance,
  Dinic == Boykov-Kolmogorov, and the flow certificate of SURVEY.md §8(c).
"""
import json
import os

import numpy as np
import pytest

import oracle
import synth

DY = [0, 0, 1, -1, 1, -1, 1, -1]
DX = [1, -1, 0, 0, 1, -1, -1, 1]
GOLD = os.path.join(os.path.dirname(__file__), "golden", "spec_examples.json")


def py_arcs(H, W, K):
    """(p, q, k) for every in-grid directed n-link p -> q = p + d_k."""
    out = []
    for y in range(H):
        for x in range(W):
            for k in range(K):
                y2, x2 = y + DY[k], x + DX[k]
                if 0 <= y2 < H and 0 <= x2 < W:
                    out.append((y * W + x, y2 * W + x2, k))
    return out


def py_brute(cs, ct, nb):
    """Independent enumeration: F* = min_S cut(S), mask* = AND of all minimisers."""
    K, H, W = nb.shape
    N = H * W
    S = (np.arange(1 << N, dtype=np.int64)[:, None] >> np.arange(N)[None, :]) & 1  # [2^N, N]
    csf, ctf = cs.reshape(-1).astype(np.int64), ct.reshape(-1).astype(np.int64)
    cut = (1 - S) @ csf + S @ ctf
    for p, q, k in py_arcs(H, W, K):
        c = int(nb[k].reshape(-1)[p])
        if c:
            cut += c * (S[:, p] * (1 - S[:, q]))
    best = cut.min()
    inter = np.all(S[cut == best] == 1, axis=0)
    return int(best), inter.reshape(H, W).astype(np.uint8)


def rand_case(rng, H, W, K, tmax=6, nmax=6, zero=0.3):
    cs, ct, nb = synth.random_caps(rng, H, W, K, tmax=tmax, nmax=nmax, zero_frac=zero, garbage=True)
    return cs[0], ct[0], nb[0]


SMALL = [(1, 1), (1, 2), (1, 5), (1, 8), (2, 2), (2, 3), (2, 5), (3, 3), (3, 4), (4, 3), (4, 4)]


@pytest.mark.parametrize("K", [4, 8])
@pytest.mark.parametrize("algo", ["dinic", "bk"])
def test_oracle_vs_python_brute_random(K, algo):
    rng = np.random.default_rng(1000 + K)
    for (H, W) in SMALL:
        for rep in range(12):
            tmax = [2, 6, 30][rep % 3]  # small caps -> many ties
            cs, ct, nb = rand_case(rng, H, W, K, tmax=tmax, nmax=tmax)
            Fb, mb = py_brute(cs, ct, nb)
            F, m = oracle.solve(cs, ct, nb, algo)
            assert F == Fb, (H, W, K, rep)
            np.testing.assert_array_equal(m, mb, err_msg=f"{H}x{W} K={K} rep={rep}")


def test_c_brute_vs_python_brute():
    rng = np.random.default_rng(7)
    for (H, W) in SMALL[:9]:
        for K in (4, 8):
            cs, ct, nb = rand_case(rng, H, W, K, tmax=3, nmax=3)
            assert oracle.brute(cs, ct, nb)[0] == py_brute(cs, ct, nb)[0]
            np.testing.assert_array_equal(oracle.brute(cs, ct, nb)[1], py_brute(cs, ct, nb)[1])


def test_spec_golden_examples():
    g = json.load(open(GOLD))
    for c in g["cases"]:
        cs, ct, nb = (np.array(c[k], np.int32) for k in ("cap_s", "cap_t", "cap_nb"))
        for algo in ("dinic", "bk"):
            F, m = oracle.solve(cs, ct, nb, algo)
            assert F == c["F"], c["cite"]
            np.testing.assert_array_equal(m, np.array(c["mask"], np.uint8), err_msg=c["cite"])
        assert py_brute(cs, ct, nb)[0] == c["F"], c["cite"]
    for c in g["energy"]:
        cs, ct, nb = (np.array(c[k], np.int32) for k in ("cap_s", "cap_t", "cap_nb"))
        assert oracle.cut_value(cs, ct, nb, np.array(c["mask"], np.uint8)) == c["cut"], c["cite"]


@pytest.mark.parametrize("K", [4, 8])
def test_closed_form_no_nlinks(K):
    """No n-links: each pixel is independent -> F = sum min(cs,ct), mask = {cs > ct}."""
    rng = np.random.default_rng(11)
    H, W = 17, 23
    cs = rng.integers(0, 50, (H, W)).astype(np.int32)
    ct = rng.integers(0, 50, (H, W)).astype(np.int32)
    nb = np.zeros((K, H, W), np.int32)
    for algo in ("dinic", "bk"):
        F, m = oracle.solve(cs, ct, nb, algo)
        assert F == int(np.minimum(cs, ct).sum())
        np.testing.assert_array_equal(m, (cs > ct).astype(np.uint8))


@pytest.mark.parametrize("K", [4, 8])
def test_closed_form_strong_coupling(K):
    """n-links larger than sum of all t-links on a connected grid: the cut never separates
    pixels -> F = min(sum cs, sum ct); mask all 1 iff sum ct < sum cs (tie -> all 0)."""
    rng = np.random.default_rng(12)
    H, W = 9, 13
    for trial in range(6):
        cs = rng.integers(0, 20, (H, W)).astype(np.int32)
        ct = rng.integers(0, 20, (H, W)).astype(np.int32)
        if trial == 5:
            ct = cs.copy()  # exact tie
        big = int(cs.sum() + ct.sum() + 1)
        nb = np.full((K, H, W), big, np.int32)
        for algo in ("dinic", "bk"):
            F, m = oracle.solve(cs, ct, nb, algo)
            assert F == min(int(cs.sum()), int(ct.sum()))
            want = 1 if ct.sum() < cs.sum() else 0
            assert np.all(m == want)


def scipy_flow_and_mask(cs, ct, nb):
    """Max flow by scipy (Dinic/Edmonds-Karp in scipy.sparse.csgraph) on the same graph,
    and the canonical mask recomputed here by BFS from s in scipy's residual."""
    from scipy.sparse import csr_matrix
    from scipy.sparse.csgraph import maximum_flow
    K, H, W = nb.shape
    N = H * W
    s, t = N, N + 1
    cap = {}

    def add(u, v, c):
        if c:
            cap[(u, v)] = cap.get((u, v), 0) + int(c)
    for v in range(N):
        add(s, v, cs.reshape(-1)[v])
        add(v, t, ct.reshape(-1)[v])
    for p, q, k in py_arcs(H, W, K):
        add(p, q, nb[k].reshape(-1)[p])
    rows = [u for (u, v) in cap] + [v for (u, v) in cap if (v, u) not in cap]
    cols = [v for (u, v) in cap] + [u for (u, v) in cap if (v, u) not in cap]
    data = [cap[(u, v)] for (u, v) in cap] + [0 for (u, v) in cap if (v, u) not in cap]
    M = csr_matrix((np.array(data, np.int32), (rows, cols)), shape=(N + 2, N + 2))
    res = maximum_flow(M, s, t)
    flow = res.flow.toarray() if hasattr(res, "flow") else res.residual.toarray()
    capm = M.toarray()
    resid = capm - flow
    seen = np.zeros(N + 2, bool)
    seen[s] = True
    stack = [s]
    while stack:
        u = stack.pop()
        for v in np.nonzero(resid[u] > 0)[0]:
            if not seen[v]:
                seen[v] = True
                stack.append(v)
    return int(res.flow_value), seen[:N].reshape(H, W).astype(np.uint8)


@pytest.mark.parametrize("K", [4, 8])
def test_oracle_vs_scipy_maxflow(K):
    rng = np.random.default_rng(21 + K)
    for (H, W) in [(6, 9), (12, 10), (15, 16)]:
        for rep in range(3):
            cs, ct, nb = rand_case(rng, H, W, K, tmax=40, nmax=25, zero=0.25)
            Fs, ms = scipy_flow_and_mask(cs, ct, nb)
            for algo in ("dinic", "bk"):
                F, m = oracle.solve(cs, ct, nb, algo)
                assert F == Fs
                np.testing.assert_array_equal(m, ms)


@pytest.mark.parametrize("K", [4, 8])
def test_c1_crops_brute_force(K):
    """C1: all 192 non-overlapping 4x4 crops of the 64x48 blob frame (crop-internal n-links
    only) -- oracle vs independent python brute force."""
    cs, ct, nb = synth.gen_host("blob", synth.BASE_SEED + 0, 0, 1, 48, 64, K)
    cs, ct, nb = cs[0], ct[0], nb[0]
    n = 0
    for y0 in range(0, 48, 4):
        for x0 in range(0, 64, 4):
            c_s, c_t = cs[y0:y0 + 4, x0:x0 + 4], ct[y0:y0 + 4, x0:x0 + 4]
            c_n = nb[:, y0:y0 + 4, x0:x0 + 4]
            Fb, mb = py_brute(c_s, c_t, c_n)
            F, m = oracle.solve(c_s, c_t, c_n, "bk" if n % 2 else "dinic")
            assert F == Fb
            np.testing.assert_array_equal(m, mb)
            n += 1
    assert n == 192


@pytest.mark.parametrize("kind,H,W,K", [("blob", 48, 64, 4), ("blob", 48, 64, 8), ("blob", 120, 160, 4),
                                        ("serpentine", 96, 128, 4), ("random", 40, 50, 8)])
def test_dinic_equals_bk_and_duality(kind, H, W, K):
    if kind == "serpentine":
        synth.set_serpentine_params(lane=8, big=1 << 20)
    if kind == "random":
        synth.set_random_params(200, 100, 30)
    cs, ct, nb = synth.gen_host(kind, synth.BASE_SEED + 1, 3, 1, H, W, K)
    cs, ct, nb = cs[0], ct[0], nb[0]
    Fd, md = oracle.solve(cs, ct, nb, "dinic")
    Fb, mb = oracle.solve(cs, ct, nb, "bk")
    assert Fd == Fb
    np.testing.assert_array_equal(md, mb)
    assert oracle.cut_value(cs, ct, nb, md) == Fd  # duality: flow value == capacity of the cut
    synth.set_serpentine_params()
    synth.set_random_params()


def test_monotonicity():
    """Raising any single capacity never lowers F."""
    rng = np.random.default_rng(31)
    for rep in range(30):
        K = 4 if rep % 2 else 8
        cs, ct, nb = rand_case(rng, 5, 6, K, tmax=10, nmax=10)
        F0 = oracle.solve(cs, ct, nb)[0]
        which = rep % 3
        y, x = rng.integers(0, 5), rng.integers(0, 6)
        cs2, ct2, nb2 = cs.copy(), ct.copy(), nb.copy()
        if which == 0:
            cs2[y, x] += rng.integers(1, 10)
        elif which == 1:
            ct2[y, x] += rng.integers(1, 10)
        else:
            nb2[rng.integers(0, K), y, x] = abs(int(nb2[0, y, x])) % 50 + 5
        assert oracle.solve(cs2, ct2, nb2)[0] >= F0


def test_tlink_normalisation_invariance():
    """Subtracting min(cs,ct) per pixel changes F by exactly sum(min) and keeps the mask
    (reading c8)."""
    cs, ct, nb = synth.gen_host("blob", synth.BASE_SEED + 2, 5, 1, 48, 64, 4)
    cs, ct, nb = cs[0], ct[0], nb[0]
    mn = np.minimum(cs, ct)
    F, m = oracle.solve(cs, ct, nb)
    F2, m2 = oracle.solve(cs - mn, ct - mn, nb)
    assert F2 == F - int(mn.sum())
    np.testing.assert_array_equal(m, m2)


def certificate_F(cs, ct, nb, f):
    """SURVEY.md §8(c) flow certificate: for an arc-feasible forward flow f [K/2,H,W],
    e = cs - ct + in - out and F(f) = sum ct - sum max(0, -e) <= F*.  Returns None if f is
    not arc-feasible."""
    K, H, W = nb.shape
    e = cs.astype(np.int64) - ct.astype(np.int64)
    for j in range(K // 2):
        k = 2 * j
        for y in range(H):
            for x in range(W):
                y2, x2 = y + DY[k], x + DX[k]
                fv = int(f[j, y, x])
                if not (0 <= y2 < H and 0 <= x2 < W):
                    if fv != 0:
                        return None
                    continue
                if fv > nb[k, y, x] or -fv > nb[k ^ 1, y2, x2]:
                    return None
                e[y, x] -= fv
                e[y2, x2] += fv
    return int(ct.astype(np.int64).sum() - np.maximum(0, -e).sum())


def test_flow_certificate_lemma():
    """Any arc-feasible flow gives F(f) <= F*, with equality for the oracle's max flow."""
    rng = np.random.default_rng(41)
    tight = 0
    for rep in range(40):
        K = 4 if rep % 2 else 8
        cs, ct, nb = rand_case(rng, 3, 4, K, tmax=8, nmax=8, zero=0.2)
        Fstar, _ = py_brute(cs, ct, nb)
        F, m, fw = oracle.solve(cs, ct, nb, "dinic", want_flow=True)
        assert certificate_F(cs, ct, nb, fw) == Fstar
        # random feasible flow
        f = np.zeros((K // 2, 3, 4), np.int64)
        for j in range(K // 2):
            k = 2 * j
            for y in range(3):
                for x in range(4):
                    y2, x2 = y + DY[k], x + DX[k]
                    if 0 <= y2 < 3 and 0 <= x2 < 4:
                        lo, hi = -int(nb[k ^ 1, y2, x2]), int(nb[k, y, x])
                        f[j, y, x] = rng.integers(lo, hi + 1)
        Ff = certificate_F(cs, ct, nb, f)
        assert Ff is not None and Ff <= Fstar
        tight += Ff == Fstar
    assert tight < 40


def test_solve_batch_threads():
    cs, ct, nb = synth.gen_host("blob", synth.BASE_SEED + 3, 0, 4, 48, 64, 4)
    F, m = oracle.solve_batch(cs, ct, nb, "bk", threads=2)
    for i in range(4):
        Fi, mi = oracle.solve(cs[i], ct[i], nb[i], "dinic")
        assert F[i] == Fi
        np.testing.assert_array_equal(m[i], mi)
