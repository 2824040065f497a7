"""Shared checkers of the GPU tests (test infrastructure): oracle comparison, the
oracle-free flow certificate and the canonical-cut recomputation of SURVEY.md §8(c)."""
import numpy as np

import oracle

DY = [0, 0, 1, -1, 1, -1, 1, -1]
DX = [1, -1, 0, 0, 1, -1, -1, 1]


def check_against_oracle(cs, ct, nb, F, mask, algo="dinic", frames=None):
    n = cs.shape[0]
    idx = range(n) if frames is None else frames
    for i in idx:
        Fo, mo = oracle.solve(cs[i], ct[i], nb[i], algo)
        assert int(F[i]) == Fo, f"frame {i}: F gpu {int(F[i])} oracle {Fo}"
        if not np.array_equal(mask[i], mo):
            bad = np.argwhere(mask[i] != mo)
            raise AssertionError(f"frame {i}: {len(bad)} mask mismatches, first {bad[:5].tolist()}")


def cut_cert(cs, ct, nb, f):
    """Oracle-free certificate: e from caps and the exported forward flow;
    F(f) = sum ct - sum max(0,-e); returns (feasible, F(f))."""
    K, H, W = nb.shape
    e = cs.astype(np.int64) - ct.astype(np.int64)
    ok = True
    for j in range(K // 2):
        k = 2 * j
        fj = f[j].astype(np.int64)
        y0, y1 = max(0, -DY[k]), H - max(0, DY[k])
        x0, x1 = max(0, -DX[k]), W - max(0, DX[k])
        src = fj[y0:y1, x0:x1]
        cfw = nb[k, y0:y1, x0:x1].astype(np.int64)
        crv = nb[k ^ 1, y0 + DY[k]:y1 + DY[k], x0 + DX[k]:x1 + DX[k]].astype(np.int64)
        ok &= bool(np.all(src <= cfw) and np.all(-src <= crv))
        e[y0:y1, x0:x1] -= src
        e[y0 + DY[k]:y1 + DY[k], x0 + DX[k]:x1 + DX[k]] += src
        # off-grid flows must be zero
        full = np.zeros_like(fj, bool)
        full[y0:y1, x0:x1] = True
        ok &= bool(np.all(fj[~full] == 0))
    return ok, int(ct.astype(np.int64).sum() - np.maximum(0, -e).sum())


def cut_torch(torch, cs, ct, nb, mask):
    """cut(S) of SURVEY.md §8(c), S = mask, written out in plain PyTorch on the device:
    sum_{v not in S} cs + sum_{v in S} ct + sum over in-grid arcs p -> q, p in S, q not in S."""
    S = mask.bool()
    n, K, H, W = nb.shape
    val = torch.where(S, ct, cs).to(torch.int64).sum(dim=(1, 2))
    for k in range(K):
        dy, dx = DY[k], DX[k]
        y0, y1 = max(0, -dy), H - max(0, dy)
        x0, x1 = max(0, -dx), W - max(0, dx)
        p = S[:, y0:y1, x0:x1]
        q = S[:, y0 + dy:y1 + dy, x0 + dx:x1 + dx]
        val += (nb[:, k, y0:y1, x0:x1].to(torch.int64) * (p & ~q)).sum(dim=(1, 2))
    return val


def residual_closure_host(cs, ct, nb, f):
    """Pixels reachable from s in the residual graph of the exported flow f:
    the closure of {e > 0} (s -> v keeps residual capacity e(v)) under n-link arcs with
    r_k(p) = c_k(p) - f(p -> p + d_k) > 0.  Plain scipy BFS (library routine), no solver code."""
    import scipy.sparse as sp
    from scipy.sparse.csgraph import breadth_first_order
    K, H, W = nb.shape
    N = H * W
    idx = np.arange(N, dtype=np.int64).reshape(H, W)
    e = cs.astype(np.int64) - ct.astype(np.int64)
    flow = {}  # flow on arc p -> p + d_k for every k, from the forward-arc flows
    for j in range(K // 2):
        k = 2 * j
        fk = np.zeros((H, W), np.int64)
        y0, y1 = max(0, -DY[k]), H - max(0, DY[k])
        x0, x1 = max(0, -DX[k]), W - max(0, DX[k])
        fk[y0:y1, x0:x1] = f[j, y0:y1, x0:x1]
        flow[k] = fk
        rv = np.zeros((H, W), np.int64)  # reverse arc q -> p carries -f(p -> q), stored at q
        rv[y0 + DY[k]:y1 + DY[k], x0 + DX[k]:x1 + DX[k]] = -fk[y0:y1, x0:x1]
        flow[k ^ 1] = rv
        e[y0:y1, x0:x1] -= fk[y0:y1, x0:x1]
        e[y0 + DY[k]:y1 + DY[k], x0 + DX[k]:x1 + DX[k]] += fk[y0:y1, x0:x1]
    rows, cols = [], []
    for k in range(K):
        y0, y1 = max(0, -DY[k]), H - max(0, DY[k])
        x0, x1 = max(0, -DX[k]), W - max(0, DX[k])
        r = nb[k, y0:y1, x0:x1].astype(np.int64) - flow[k][y0:y1, x0:x1]
        open_ = r > 0
        rows.append(idx[y0:y1, x0:x1][open_])
        cols.append(idx[y0 + DY[k]:y1 + DY[k], x0 + DX[k]:x1 + DX[k]][open_])
    src = np.flatnonzero(e.ravel() > 0)  # super-source N -> every excess node
    rows.append(np.full(src.size, N, np.int64))
    cols.append(src)
    r_ = np.concatenate(rows)
    c_ = np.concatenate(cols)
    G = sp.csr_matrix((np.ones(r_.size, np.int8), (r_, c_)), shape=(N + 1, N + 1))
    order = breadth_first_order(G, N, directed=True, return_predecessors=False)
    m = np.zeros(N + 1, np.uint8)
    m[order] = 1
    return m[:N].reshape(H, W)
