"""NumPy executor of a host-only HddPlan (test infrastructure).

Runs the exact algebra of the CUDA kernels (csrc/hdd_kernels.cu) on the CPU,
driven only by the plan tables the C ABI exports (hdd_plan_*_info,
hdd_leaf_template).  It checks the C++ plan builder — index sets, gather
maps, column routing, in-leaf births — against the oracle without a GPU.
"""
from __future__ import annotations

import ctypes as C

import numpy as np
import scipy.linalg

from paper_1708_02207_b200 import _lib

LEAF = 16
P1 = np.zeros((4, 4))
P1[np.ix_([0, 1, 3], [0, 1, 3])] = 0.5 * np.array([[1, -1, 0], [-1, 2, -1], [0, -1, 1.0]])
P2 = np.zeros((4, 4))
P2[np.ix_([0, 3, 2], [0, 3, 2])] = 0.5 * np.array([[1, 0, -1], [0, 1, -1], [-1, -1, 2.0]])


def _arr(ptr, n, dtype):
    if n == 0:
        return np.zeros(0, dtype=dtype)
    return np.ctypeslib.as_array(ptr, shape=(n,)).astype(dtype).copy()


def leaf_template():
    L = _lib.lib()
    out = []
    for r in range(8):
        K, k, ng = C.c_int32(), C.c_int32(), C.c_int32()
        m1, m2 = _lib._i32p(), _lib._i32p()
        assert L.hdd_leaf_template(r, C.byref(K), C.byref(k), C.byref(ng), C.byref(m1), C.byref(m2)) == 0
        out.append((K.value, k.value, ng.value, _arr(m1, K.value, int), _arr(m2, K.value, int)))
    return out


def origin(r, q):
    x = y = 0
    w = h = LEAF
    for lev in range(r):
        b = (q >> (r - 1 - lev)) & 1
        if lev % 2 == 0:
            w //= 2
            x += w * b
        else:
            h //= 2
            y += h * b
    return x, y


def eliminate(At, Rt, sig, k, factors=None):
    """Bordered Schur complement: returns (Psi, R, sigma); `factors` (a list)
    receives (L, W, v) for the primal top-down pass."""
    ng = At.shape[0] - k
    if ng == 0:
        return At[:k, :k].copy(), Rt[:k].copy(), sig.copy()
    Lc = scipy.linalg.cholesky(At[k:, k:], lower=True)
    W = scipy.linalg.solve_triangular(Lc, At[k:, :k], lower=True)
    V = scipy.linalg.solve_triangular(Lc, Rt[k:], lower=True)
    Psi = At[:k, :k] - W.T @ W
    R = Rt[:k] - W.T @ V
    s = sig.copy()
    s[1:] += V[:, 0] @ V[:, 1:]
    if factors is not None:
        factors.append((Lc, W, V[:, 0]))
    return Psi, R, s


def run(plan, level, kappa, f=None):
    L = _lib.lib()
    info = _lib.HddPlanInfo()
    assert L.hdd_plan_info(plan.handle, C.byref(info)) == 0
    N = 1 << level
    m = N + 1
    h = 1.0 / N
    f = np.ones(m * m) if f is None else f
    tmpl = leaf_template()
    h2_6 = h * h / 6.0
    loadpat = np.array([h2_6 + h2_6, h2_6, h2_6, h2_6 + h2_6])
    meanpat = np.array([1 / 3, 1 / 6, 1 / 6, 1 / 3])
    leaf_out = []
    for li in range(info.n_leaves):
        lf = _lib.HddLeafInfo()
        assert L.hdd_plan_leaf_info(plan.handle, li, C.byref(lf)) == 0
        nc = lf.ncols
        birth = _arr(lf.birth, 3 * nc, int).reshape(nc, 3)
        ctype = _arr(lf.ccode, nc, int)
        assert ctype[0] == 0 and (nc > 1 and ctype[1] == 1) == bool(lf.has_mean)
        sub = [(c, ctype[c] & 31, (ctype[c] >> 5) & 31, (ctype[c] >> 10) & 31, (ctype[c] >> 15) & 31)
               for c in range(nc) if ctype[c] >= 1 << 24]       # means over sub-leaf nodes
        coef = np.where(ctype == 1, 0.5, 1.0)
        # cells
        level_nodes = []
        for q in range(256):
            x, y = origin(8, q)
            i, j = lf.i0 + x, lf.j0 + y
            t = 2 * (i * N + j)
            psi = kappa[t] * P1 + kappa[t + 1] * P2
            R = np.zeros((4, nc))
            nodes = [j * m + i, j * m + i + 1, (j + 1) * m + i, (j + 1) * m + i + 1]
            R[:, 0] = loadpat * f[nodes]
            if lf.has_mean:
                R[:, 1] = meanpat
            for c, i0, i1, j0, j1 in sub:
                if i0 <= x < i1 and j0 <= y < j1:
                    R[:, c] = loadpat
            level_nodes.append((psi, R, np.zeros(nc)))
        for r in range(7, -1, -1):
            K, k, ng, m1, m2 = tmpl[r]
            new = []
            for q in range(1 << r):
                At = np.zeros((K, K))
                Rt = np.zeros((K, nc))
                sg = np.zeros(nc)
                for mp, son in ((m1, level_nodes[2 * q]), (m2, level_nodes[2 * q + 1])):
                    sel = np.flatnonzero(mp >= 0)
                    At[np.ix_(sel, sel)] += son[0][np.ix_(mp[sel], mp[sel])]
                    Rt[sel] += son[1][mp[sel]] * coef
                    sg += son[2] * coef
                for c in range(nc):
                    if birth[c, 0] == r and birth[c, 1] == q:
                        Rt[k + birth[c, 2], c] += 1.0
                new.append(eliminate(At, Rt, sg, k))
            level_nodes = new
        psi, R, sg = level_nodes[0]
        if lf.gperim:
            # known boundary values: load rows r -= Psi_{.,D} g_D, functionals sigma += R_D^T g_D
            gp = _arr(lf.gperim, 64, float)
            R = R.copy()
            sg = sg.copy()
            R[:, 0] -= psi @ gp
            sg[1:] += gp @ R[:, 1:]
        for c, i0, i1, j0, j1 in sub:
            R[:, c] /= (i1 - i0) * (j1 - j0) * h * h
            sg[c] /= (i1 - i0) * (j1 - j0) * h * h
        leaf_out.append((psi, R, sg))
    upper_out = {}

    def son_out(s):
        return upper_out[s] if s >= 0 else leaf_out[-1 - s]

    nodes = []
    for u in range(info.n_upper):
        nd = _lib.HddNodeInfo()
        assert L.hdd_plan_node_info(plan.handle, u, C.byref(nd)) == 0
        nodes.append(nd)
    facs = {}
    for u, nd in enumerate(nodes):   # plan order: deepest first
        k, ng, nc = nd.k, nd.ng, nd.nc
        K = k + ng
        gmap = _arr(nd.gmap, 2 * K, int).reshape(2, K)
        csrc = _arr(nd.csrc, 2 * nc, int).reshape(nc, 2)
        ccoef = _arr(nd.ccoef, 2 * nc, float).reshape(nc, 2)
        cb = _arr(nd.cbirth, nc, int)
        At = np.zeros((K, K))
        Rt = np.zeros((K, nc))
        sg = np.zeros(nc)
        for si in range(2):
            psi, R, s = son_out(nd.son[si])
            mp = gmap[si]
            sel = np.flatnonzero(mp >= 0)
            At[np.ix_(sel, sel)] += psi[np.ix_(mp[sel], mp[sel])]
            for c in range(nc):
                if csrc[c, si] >= 0:
                    Rt[sel, c] += ccoef[c, si] * R[mp[sel], csrc[c, si]]
                    sg[c] += ccoef[c, si] * s[csrc[c, si]]
        for c in range(nc):
            if cb[c] >= 0:
                Rt[k + cb[c], c] += 1.0
        fl_ = []
        upper_out[u] = eliminate(At, Rt, sg, k, fl_)
        facs[u] = fl_[0] if fl_ else None
    root_sig = upper_out[info.n_upper - 1][2] if info.n_upper else leaf_out[0][2]
    # primal top-down (root first = reverse plan order): u_K = [u_B | u_gamma]
    uK = {}
    parent_of = {}
    for u, nd in enumerate(nodes):
        for si in range(2):
            parent_of[nd.son[si]] = (u, si)
    for u in range(info.n_upper - 1, -1, -1):
        nd = nodes[u]
        k, ng = nd.k, nd.ng
        if u in parent_of:
            pu, si = parent_of[u]
            pg = _arr(nodes[pu].gmap, 2 * (nodes[pu].k + nodes[pu].ng), int).reshape(2, -1)[si]
            uB = np.zeros(k)
            sel = np.flatnonzero(pg >= 0)
            uB[pg[sel]] = uK[pu][sel]
        else:
            uB = np.zeros(k)
        Lc, W, v = facs[u]
        ug = scipy.linalg.solve_triangular(Lc.T, v - W @ uB, lower=False)
        uK[u] = np.concatenate([uB, ug])
    S = np.empty(info.n_obs)
    for o in range(info.n_obs):
        ob = _lib.HddObsInfo()
        assert L.hdd_plan_obs_info(plan.handle, o, C.byref(ob)) == 0
        if ob.kind == 0:
            S[o] = root_sig[ob.col]
        elif ob.kind == 1:
            S[o] = ob.value
        elif ob.kind == 3:
            S[o] = uK[ob.node][nodes[ob.node].k + ob.col]
        else:
            leaf = -1 - ob.node if ob.node < 0 else ob.node
            pu, si = parent_of[-1 - leaf]
            pg = _arr(nodes[pu].gmap, 2 * (nodes[pu].k + nodes[pu].ng), int).reshape(2, -1)[si]
            uB = np.zeros(64)
            sel = np.flatnonzero(pg >= 0)
            uB[pg[sel]] = uK[pu][sel]
            psi, R, sg = leaf_out[leaf]
            S[o] = R[:, ob.col] @ uB + sg[ob.col]
    return S, leaf_out, upper_out
