"""CPU oracle for the periodic FMM + HI electrostatics path.

TEST INFRASTRUCTURE — NOT PART OF THE PRODUCT.  Only ``tests/``,
``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` / reference
arm may import this module, and only as the checker or as the timed CPU
baseline; the GPU path never calls it.

It restates, in complex128 numpy, the algorithm of the reference package
``lambdafmm`` 0.1.0 (paths relative to /root/reference/pkg/src/lambdafmm):
solid harmonics and translation operators (fmm/harmonics.py), the uniform
periodic octree (fmm/octree.py), the lattice operator and surface term
(fmm/lattice.py), the solve / spatial-force pipeline (fmm/solver.py) and
the HI correction + assembly (corrections.py, weights.py, system.py).
The vectorisation is its own (padded leaf blocks for P2P, particle-batched
P2M/L2P, parity-grouped M2L) but every formula follows the cited lines.

Parity pin: ``tests/golden/*.npz`` were produced by running the reference
itself (tests/golden/make_golden.py); tests/test_oracle.py checks this
oracle against them and against the reference's known-answer values.
"""

import math
from functools import lru_cache

import numpy as np

DIPOLE_ETA = -1.0  # lattice.py:41


# ----------------------------------------------------------- harmonics ----
def ncoef(p):
    return (p + 1) ** 2


def cidx(l, m):
    return l * l + l + m  # harmonics.py:37


@lru_cache(maxsize=None)
def lm_tables(p):
    ls = np.repeat(np.arange(p + 1), 2 * np.arange(p + 1) + 1)
    ms = np.concatenate([np.arange(-l, l + 1) for l in range(p + 1)])
    return ls, ms


def regular(xyz, p):
    """R_l^m(r) = P_l^m r^l e^{im phi}/(l+m)!  by recurrence (harmonics.py:58-77)."""
    xyz = np.atleast_2d(np.asarray(xyz, dtype=np.float64))
    x, y, z = xyz[:, 0], xyz[:, 1], xyz[:, 2]
    u = x + 1j * y
    rr = x * x + y * y + z * z
    out = np.zeros((xyz.shape[0], ncoef(p)), np.complex128)
    diag = np.ones(xyz.shape[0], np.complex128)
    for m in range(p + 1):
        if m:
            diag = diag * u / (2.0 * m)
        out[:, cidx(m, m)] = diag
        if m < p:
            out[:, cidx(m + 1, m)] = z * diag
        for l in range(m + 2, p + 1):
            out[:, cidx(l, m)] = ((2 * l - 1) * z * out[:, cidx(l - 1, m)]
                                  - rr * out[:, cidx(l - 2, m)]) / ((l + m) * (l - m))
    _fill_negative(out, p)
    return out


def irregular(xyz, p):
    """I_l^m(r) = (l-m)! P_l^m e^{im phi}/r^(l+1)  (harmonics.py:80-103)."""
    xyz = np.atleast_2d(np.asarray(xyz, dtype=np.float64))
    x, y, z = xyz[:, 0], xyz[:, 1], xyz[:, 2]
    u = x + 1j * y
    inv2 = 1.0 / (x * x + y * y + z * z)
    out = np.zeros((xyz.shape[0], ncoef(p)), np.complex128)
    diag = np.sqrt(inv2).astype(np.complex128)
    for m in range(p + 1):
        if m:
            diag = (2 * m - 1) * diag * u * inv2
        out[:, cidx(m, m)] = diag
        if m < p:
            out[:, cidx(m + 1, m)] = (2 * m + 1) * z * diag * inv2
        for l in range(m + 2, p + 1):
            out[:, cidx(l, m)] = ((2 * l - 1) * z * out[:, cidx(l - 1, m)]
                                  - ((l - 1) ** 2 - m * m) * out[:, cidx(l - 2, m)]) * inv2
    _fill_negative(out, p)
    return out


def _fill_negative(out, p):
    # X_l^{-m} = (-1)^m conj(X_l^m)  (harmonics.py:3-8)
    for l in range(1, p + 1):
        for m in range(1, l + 1):
            out[:, cidx(l, -m)] = (-1) ** m * np.conj(out[:, cidx(l, m)])


def regular_grad(xyz, p):
    """Cartesian gradient of R_l^m via the R_{l-1} ladder (harmonics.py:106-130)."""
    r = regular(xyz, p)
    ls, ms = lm_tables(p)
    g = np.zeros(r.shape + (3,), np.complex128)
    for dm, col in ((-1, "a"), (1, "b"), (0, "c")):
        lt, mt = ls - 1, ms + dm
        ok = (lt >= 0) & (np.abs(mt) <= lt)
        src = np.where(ok, lt * lt + lt + mt, 0)
        v = np.where(ok[None, :], r[:, src], 0.0)
        if col == "a":
            g[..., 0] += 0.5 * v
            g[..., 1] += 0.5j * v
        elif col == "b":
            g[..., 0] -= 0.5 * v
            g[..., 1] += 0.5j * v
        else:
            g[..., 2] = v
    return g


@lru_cache(maxsize=None)
def _shift_map(p):
    ls, ms = lm_tables(p)
    dl = ls[:, None] - ls[None, :]
    dm = ms[:, None] - ms[None, :]
    ok = (dl >= 0) & (np.abs(dm) <= dl)
    return np.where(ok, dl * dl + dl + dm, 0), ok


@lru_cache(maxsize=None)
def _m2l_gather(p):
    ls, ms = lm_tables(p)
    L = ls[:, None] + ls[None, :]
    M = -(ms[:, None] + ms[None, :])
    sign = np.where((ls[None, :] + ms[:, None] + ms[None, :]) % 2 == 0, 1.0, -1.0)
    return L * L + L + M, sign


def m2m_op(d, p):
    """M_new = A M_old for c_new = c_old + d (harmonics.py:155-159)."""
    src, ok = _shift_map(p)
    rv = regular(-np.asarray(d, float)[None, :], p)[0]
    return np.where(ok, rv[src], 0.0)


def l2l_op(d, p):
    """L_new = C L_old for c_new = c_old + d (harmonics.py:162-166)."""
    src, ok = _shift_map(p)
    rv = regular(np.asarray(d, float)[None, :], p)[0]
    return np.where(ok, rv[src], 0.0).T


def m2l_from_iv(iv, p):
    """B from I(-d) at order 2p (harmonics.py:196-203)."""
    src, sign = _m2l_gather(p)
    return sign * iv[..., src]


# -------------------------------------------------------------- octree ----
NB_OFF = np.array([(a, b, c) for a in (-1, 0, 1) for b in (-1, 0, 1) for c in (-1, 0, 1)], np.int64)
_C3 = np.array([(a, b, c) for a in range(-3, 4) for b in range(-3, 4) for c in range(-3, 4)], np.int64)
M2L_OFF = _C3[np.abs(_C3).max(1) >= 2]  # (316,3) octree.py:31
OCT = np.array([(a, b, c) for a in (0, 1) for b in (0, 1) for c in (0, 1)], np.int64)


def grid_of(n):
    i = np.arange(n ** 3, dtype=np.int64)
    return np.stack([i // (n * n), (i // n) % n, i % n], 1)


def flat(g, n):
    return (g[..., 0] * n + g[..., 1]) * n + g[..., 2]


def wrap(pos, box):
    """np.mod wrap, exact box multiples -> 0 (system.py:103-108)."""
    w = np.mod(np.asarray(pos, np.float64), box)
    w[w >= box] = 0.0
    return w


def m2l_pairs(level):
    """Per M2L_OFFSETS row: targets whose parity admits the offset and their
    wrapped sources (octree.py:35-38, :96-111)."""
    n = 2 ** level
    g = grid_of(n)
    par = g & 1
    out = []
    for row, o in enumerate(M2L_OFF):
        ok = np.all((-2 - par <= o) & (o <= 3 - par), axis=1)
        t = np.flatnonzero(ok)
        if t.size:
            out.append((row, t, flat(np.mod(g[t] + o, n), n)))
    return out


def build_tree(pos, box, depth):
    """Canonical order + CSR + periodic neighbours (octree.py:114-163)."""
    pos = np.atleast_2d(np.asarray(pos, np.float64))
    n = 2 ** depth
    size = box / n
    cell = np.clip((pos / size).astype(np.int64), 0, n - 1)
    leaf = flat(cell, n)
    perm = np.lexsort((pos[:, 2], pos[:, 1], pos[:, 0], leaf))
    inv = np.empty_like(perm)
    inv[perm] = np.arange(perm.size)
    start = np.zeros(n ** 3 + 1, np.int64)
    np.cumsum(np.bincount(leaf, minlength=n ** 3), out=start[1:])
    raw = grid_of(n)[:, None, :] + NB_OFF[None]
    shift = np.floor_divide(raw, n)
    nb = flat(raw - shift * n, n)
    return dict(perm=perm, inv_perm=inv, positions=pos[perm], leaf_of_particle=leaf[perm], leaf_start=start,
                nb_box=nb, nb_shift=shift, depth=depth, box=float(box), size=size)


# ------------------------------------------------------------- lattice ----
def image_vectors(smin, smax):
    a = np.arange(-smax, smax + 1)
    g = np.stack(np.meshgrid(a, a, a, indexing="ij"), -1).reshape(-1, 3)
    nrm = np.abs(g).max(1)
    return g[(nrm >= smin) & (nrm <= smax)].astype(np.float64)


def _symmetrise(t):
    return 0.5 * (t + t.T)


@lru_cache(maxsize=8)
def lattice_shells(p, cap):
    """Exact finite-shell far-image operator (lattice.py:109-121)."""
    v = image_vectors(2, cap)
    iv = np.zeros(ncoef(2 * p), np.complex128)
    for lo in range(0, v.shape[0], 4096):
        iv += irregular(v[lo:lo + 4096], 2 * p).sum(0)
    return _symmetrise(m2l_from_iv(iv, p))


@lru_cache(maxsize=8)
def lattice_converged(p, steps=24):
    """Factor-3 telescoped infinite lattice (lattice.py:124-155)."""
    ls, _ = lm_tables(p)
    t_ring = m2l_from_iv(irregular(image_vectors(2, 4), 2 * p).sum(0), p)
    src, ok = _shift_map(p)
    rv = regular(image_vectors(0, 1), p).sum(0)
    s_hat = (3.0 ** -ls)[:, None] * np.where(ok, rv[src], 0.0)
    acc = np.zeros((ncoef(p), ncoef(p)), np.complex128)
    b = np.eye(ncoef(p), dtype=np.complex128)
    for k in range(steps):
        acc += (3.0 ** (-k * (ls + 1.0)))[:, None] * (t_ring @ b)
        if k + 1 < steps:
            b = s_hat @ b
    acc[(ls[:, None] + ls[None, :]) < 4] = 0.0
    return _symmetrise(acc)


def lattice_scaled(unit, p, box):
    ls, _ = lm_tables(p)
    return (box ** -(ls + 1.0))[:, None] * unit * (box ** -ls.astype(float))[None, :]


def lattice_matrix(cfg, box):
    if cfg["lattice_mode"] == "converged":
        return lattice_scaled(lattice_converged(cfg["p"]), cfg["p"], box)
    if cfg["lattice_mode"] == "shells":
        return lattice_scaled(lattice_shells(cfg["p"], cfg["shell_cap"]), cfg["p"], box)
    return None


# ------------------------------------------------------------ near field ----
try:  # the reference accelerates the same loop with numba (solver.py:30-33, :164-195)
    import numba as _nb
except ImportError:  # pragma: no cover
    _nb = None

if _nb is not None:

    @_nb.njit(parallel=True, cache=False)
    def _p2p_numba(pos, start, nb_box, shift_len, q, rows, targets, grad, out, gout):
        nk = q.shape[1]
        for ti in _nb.prange(targets.shape[0]):
            b = targets[ti]
            t0, t1 = start[b], start[b + 1]
            for t in rows:
                s = nb_box[b, t]
                s0, s1 = start[s], start[s + 1]
                sx, sy, sz = shift_len[b, t, 0], shift_len[b, t, 1], shift_len[b, t, 2]
                home = t == 13
                for i in range(t0, t1):
                    xi, yi, zi = pos[i, 0], pos[i, 1], pos[i, 2]
                    for j in range(s0, s1):
                        if home and j == i:
                            continue
                        dx = xi - pos[j, 0] - sx
                        dy = yi - pos[j, 1] - sy
                        dz = zi - pos[j, 2] - sz
                        inv = 1.0 / np.sqrt(dx * dx + dy * dy + dz * dz)
                        for k in range(nk):
                            out[i, k] += q[j, k] * inv
                        if grad:
                            c = -q[j, 0] * inv * inv * inv
                            gout[i, 0] += c * dx
                            gout[i, 1] += c * dy
                            gout[i, 2] += c * dz


def near_field(tree, q, periodic=True, grad=False, leaves=None):
    """27-image direct sums (solver.py:126-224): V_near (N,K) and optionally
    grad V_near (N,3) for column 0, canonical order.  `leaves` restricts the
    targets (timing samples only).  Parallel numba loop over target leaves
    (each leaf's sums run serially, so results do not depend on threads)."""
    pos = tree["positions"]
    box = tree["box"]
    nleaf = tree["leaf_start"].size - 1
    v = np.zeros((pos.shape[0], q.shape[1]))
    g = np.zeros((pos.shape[0], 3))
    rows = np.arange(27) if periodic else np.array([13])
    targets = np.arange(nleaf) if leaves is None else np.asarray(leaves, np.int64)
    if _nb is not None:
        _p2p_numba(pos, tree["leaf_start"], tree["nb_box"], (tree["nb_shift"] * box).astype(np.float64),
                   np.ascontiguousarray(q, dtype=np.float64), rows, targets, bool(grad), v, g)
        return v, (g if grad else None)
    start = tree["leaf_start"]
    for b in targets:  # plain numpy fallback (solver.py:144-161)
        t0, t1 = start[b], start[b + 1]
        if t1 == t0:
            continue
        for t in rows:
            s = tree["nb_box"][b, t]
            s0, s1 = start[s], start[s + 1]
            if s1 == s0:
                continue
            d = pos[t0:t1, None, :] - (pos[None, s0:s1, :] + tree["nb_shift"][b, t] * box)
            r2 = (d * d).sum(-1)
            if t == 13:
                np.fill_diagonal(r2, np.inf)
            inv = 1.0 / np.sqrt(r2)
            v[t0:t1] += inv @ q[s0:s1]
            if grad:
                g[t0:t1] += np.einsum("tsd,ts,s->td", d, -inv ** 3, q[s0:s1, 0])
    return v, (g if grad else None)


# ------------------------------------------------------------- far field ----
def leaf_centers(tree):
    n = 2 ** tree["depth"]
    return (grid_of(n) + 0.5) * tree["size"]


def upward(tree, q, p, leaves=None):
    """Leaf P2M then M2M to the root (solver.py:227-259); list over levels of
    (nc, nbox, K) complex."""
    d = tree["depth"]
    nc = ncoef(p)
    nk = q.shape[1]
    start = tree["leaf_start"]
    lof = tree["leaf_of_particle"]
    cen = leaf_centers(tree)
    mult = [None] * (d + 1)
    m = np.zeros((nc, 8 ** d, nk), np.complex128)
    sel = np.arange(tree["positions"].shape[0])
    if leaves is not None:
        sel = np.concatenate([np.arange(start[b], start[b + 1]) for b in leaves])
    for c0 in range(0, sel.size, 65536):
        ii = sel[c0:c0 + 65536]
        r = regular(tree["positions"][ii] - cen[lof[ii]], p)  # (n, nc)
        contrib = r[:, :, None] * q[ii][:, None, :]
        # particles are leaf-sorted: segment sums per leaf
        lv = lof[ii]
        cut = np.flatnonzero(np.diff(lv)) + 1
        seg = np.add.reduceat(contrib, np.concatenate([[0], cut]), axis=0)
        m[:, lv[np.concatenate([[0], cut])], :] += np.transpose(seg, (1, 0, 2))
    mult[d] = m
    for l in range(d - 1, -1, -1):
        child_size = tree["box"] / 2 ** (l + 1)
        n = 2 ** l
        g = grid_of(n)
        mp = np.zeros((nc, n ** 3, nk), np.complex128)
        for o in range(8):
            op = m2m_op((0.5 - OCT[o]) * child_size, p)
            ci = flat(2 * g + OCT[o], 2 * n)
            mp += (op @ mult[l + 1][:, ci, :].reshape(nc, -1)).reshape(mp.shape)
        mult[l] = mp
    return mult


def m2l_level_ops(p, size):
    """Per-level operator table: irregular vectors of the 316 offsets at the
    level scale (solver.py:120-123) gathered into B matrices (harmonics.py:196)."""
    iv = irregular(M2L_OFF * size, 2 * p)
    return [m2l_from_iv(iv[row], p) for row in range(M2L_OFF.shape[0])]


def downward(tree, mult, p, root_local, boxes_fraction=None, ops=None, pairs=None):
    """L2L + offset-grouped M2L per level (solver.py:262-291)."""
    d = tree["depth"]
    nc = ncoef(p)
    nk = mult[0].shape[2]
    loc = [None] * (d + 1)
    loc[0] = np.zeros((nc, 1, nk), np.complex128) if root_local is None else root_local.reshape(nc, 1, nk)
    for l in range(1, d + 1):
        n = 2 ** l
        size = tree["box"] / n
        g = grid_of(n)
        cur = np.zeros((nc, n ** 3, nk), np.complex128)
        pg = grid_of(n // 2)
        for o in range(8):
            op = l2l_op((OCT[o] - 0.5) * size, p)
            ci = flat(2 * pg + OCT[o], n)
            cur[:, ci, :] = (op @ loc[l - 1].reshape(nc, -1)).reshape(nc, -1, nk)
        lops = ops[l] if ops is not None else m2l_level_ops(p, size)
        lim = None if boxes_fraction is None else max(1, int(math.ceil(boxes_fraction * n ** 3)))
        for row, t, s in (pairs[l] if pairs is not None else m2l_pairs(l)):
            if lim is not None:
                keep = t < lim
                t, s = t[keep], s[keep]
                if t.size == 0:
                    continue
            op = lops[row]
            cur[:, t, :] += (op @ mult[l][:, s, :].reshape(nc, -1)).reshape(nc, t.size, nk)
        loc[l] = cur
    return loc


def evaluate(tree, loc, p, grad=False, leaves=None):
    """L2P (+gradient) at the particles (solver.py:294-324)."""
    d = tree["depth"]
    cen = leaf_centers(tree)
    lof = tree["leaf_of_particle"]
    start = tree["leaf_start"]
    npart = tree["positions"].shape[0]
    nk = loc[d].shape[2]
    v = np.zeros((npart, nk))
    g = np.zeros((npart, 3)) if grad else None
    sel = np.arange(npart)
    if leaves is not None:
        sel = np.concatenate([np.arange(start[b], start[b + 1]) for b in leaves])
    for c0 in range(0, sel.size, 65536):
        ii = sel[c0:c0 + 65536]
        disp = tree["positions"][ii] - cen[lof[ii]]
        coeff = loc[d][:, lof[ii], :]  # (nc, n, K)
        r = regular(disp, p)
        v[ii] = np.real(np.einsum("nc,cnk->nk", r, coeff))
        if grad:
            gr = regular_grad(disp, p)
            g[ii] = np.real(np.einsum("ncd,cn->nd", gr, coeff[:, :, 0]))
    return v, g


# -------------------------------------------------------------- solve ----
def default_config(**kw):
    cfg = dict(p=8, depth=2, lattice_mode="converged", shell_cap=8, dipole=True, periodic_near=True,
               intra_site_images="full")
    cfg.update(kw)
    return cfg


def solve(positions, charges, box, cfg, forces=False):
    """PeriodicSolver(...).solve(q) (+ spatial_forces) in one function
    (solver.py:330-427).  Returns a dict of input-order arrays."""
    pos = wrap(np.atleast_2d(positions), box)
    tree = build_tree(pos, box, cfg["depth"])
    q = np.asarray(charges, np.float64)
    single = q.ndim == 1
    q2 = q[:, None] if single else q
    qs = q2[tree["perm"]]
    p = cfg["p"]
    vn, gn = near_field(tree, qs, cfg["periodic_near"], grad=forces)
    mult = upward(tree, qs, p)
    lat = lattice_matrix(cfg, box)
    root_local = None if lat is None else lat @ mult[0][:, 0, :]
    loc = downward(tree, mult, p, root_local)
    vf, gf = evaluate(tree, loc, p, grad=forces)
    disp = tree["positions"] - 0.5 * box
    dvec = disp.T @ qs
    gam = 2.0 * math.pi / (3.0 * box ** 3)
    if cfg["dipole"]:
        vd = 2.0 * DIPOLE_ETA * gam * (disp @ dvec)
        ed = DIPOLE_ETA * gam * (dvec * dvec).sum(0)
    else:
        vd = np.zeros_like(vn)
        ed = np.zeros(qs.shape[1])
    en = 0.5 * np.array([math.fsum((qs[:, k] * vn[:, k]).tolist()) for k in range(qs.shape[1])])
    ef = 0.5 * np.array([math.fsum((qs[:, k] * vf[:, k]).tolist()) for k in range(qs.shape[1])])
    inv = tree["inv_perm"]

    def back(a):
        a = a[inv]
        return a[:, 0] if single else a

    def sc(a):
        return a[0] if single else a

    out = dict(potentials=back(vn + vf + vd), near=back(vn), far=back(vf), dip=back(vd),
               energy=sc(en + ef + ed), near_energy=sc(en), far_energy=sc(ef), dipole_energy=sc(ed),
               root_multipole=mult[0][:, 0, 0] if single else mult[0][:, 0, :],
               dipole_vector=dvec[:, 0] if single else dvec,
               total_charge=sc(np.array([math.fsum(qs[:, k].tolist()) for k in range(qs.shape[1])])),
               tree=tree, lattice=lat)
    if forces:
        f = -qs[:, :1] * (gn + gf)
        if cfg["dipole"]:
            f += -2.0 * DIPOLE_ETA * gam * qs[:, :1] * dvec[None, :, 0]
        out["forces"] = f[inv]
    return out


# ------------------------------------------------------------------ HI ----
def weights(lams):
    """expand_weights (weights.py:54-60): lambda_0 on the LSB."""
    w = np.ones(1)
    for lam in lams:
        w = np.concatenate([w * (1.0 - lam), w * lam])
    return w


def weight_grads(lams):
    """weight_gradient_matrix (weights.py:63-85)."""
    rows = []
    for k in range(len(lams)):
        g = np.ones(1)
        for i, lam in enumerate(lams):
            g = np.concatenate([-g, g]) if i == k else np.concatenate([g * (1.0 - lam), g * lam])
        rows.append(g)
    return np.stack(rows)


def near_kernel(sp, box, images="full"):
    """corrections.near_kernel (corrections.py:46-70)."""
    disp = sp[:, None, :] - sp[None, :, :]
    if images == "minimum":
        d = disp - box * np.round(disp / box)
        r = np.sqrt((d * d).sum(-1))
        np.fill_diagonal(r, np.inf)
        return 1.0 / r
    k = np.zeros((sp.shape[0],) * 2)
    for nvec in image_vectors(0, 1):
        d = disp + nvec * box
        r = np.sqrt((d * d).sum(-1))
        if not nvec.any():
            np.fill_diagonal(r, np.inf)
        k += 1.0 / r
    return k


def lattice_kernel(sp, box, lat, p):
    """corrections.lattice_kernel (corrections.py:73-77)."""
    rv = regular(sp - 0.5 * box, p)
    return np.real(rv @ lat @ rv.T)


def hi(positions, charges, box, sites, lam_values, cfg, mode="hi", potentials=None, solve_out=None):
    """hi_energy_and_forces (corrections.py:252-274) on plain arrays.

    sites: list of (indices, form_charges (nf, ns)).  Returns dict with
    energy, forces (list), per-site c_p2p / c_lattice / c_dipole / blend."""
    q = np.array(charges, np.float64, copy=True)
    for (idx, forms), lams in zip(sites, lam_values):
        q[idx] = weights(lams) @ forms  # scale_charges (system.py:185-197)
    res = solve_out if solve_out is not None else solve(positions, q, box, cfg)
    v = res["potentials"] if potentials is None else potentials
    lat = res["lattice"]
    gam = 2.0 * math.pi / (3.0 * box ** 3)
    out = dict(forces=[], c_p2p=[], c_lattice=[], c_dipole=[], blend=[], offset=[], solve=res, q_tilde=q)
    for (idx, forms), lams in zip(sites, lam_values):
        w = weights(lams)
        gmat = weight_grads(lams)
        sp = np.asarray(positions, np.float64)[idx]
        qt = w @ forms
        half = qt[None, :] - 0.5 * forms
        dev = qt[None, :] - forms
        s_rho = forms @ v[idx]
        if mode == "qi":
            out["forces"].append(-(gmat @ s_rho))
            continue
        full = cfg["intra_site_images"] == "full"
        kern = near_kernel(sp, box, "full" if full else "minimum")
        cp = np.einsum("fs,st,ft->f", forms, kern, half)
        eb = 0.5 * float(qt @ kern @ qt)
        if full and lat is not None:
            gk = lattice_kernel(sp, box, lat, cfg["p"])
            cl = np.einsum("fs,st,ft->f", forms, gk, half)
            eb += 0.5 * float(qt @ gk @ qt)
        else:
            cl = np.zeros(forms.shape[0])
        if full and cfg["dipole"]:
            dd = dev @ (sp - 0.5 * box)
            cd = -DIPOLE_ETA * gam * (dd * dd).sum(1)
        else:
            cd = np.zeros(forms.shape[0])
        ct = cp + cl + cd
        out["forces"].append(-(gmat @ (s_rho - ct)))
        out["c_p2p"].append(cp)
        out["c_lattice"].append(cl)
        out["c_dipole"].append(cd)
        out["blend"].append(eb)
        out["offset"].append(eb - float(w @ ct))
    e = float(res["energy"])
    out["energy"] = e if mode == "qi" else e + math.fsum(out["offset"])
    return out


def hi_site_forces(positions, box, sites, lam_values, cfg, lat):
    """-grad_r Delta E_site of every site atom (A, 3), site-table order.

    Delta E_site = e(q~) - sum_rho w_rho C_rho (corrections.py:141-143,
    :179-183) with C_rho = Q_rho (K + G)(q~ - Q_rho/2) + c_dip_rho
    (:157-193) is a function of the site's own atom positions only; the
    reference has no spatial gradient of it (its spatial forces are
    spatial_forces(q~), solver.py:407-427).  Analytic gradient of the same
    pieces: near_kernel (:46-70), lattice_kernel (:73-77) through
    harmonics.regular_grad (harmonics.py:119-130), c_dipole (:112-124).
    Pinned against the reference by central differences of its per-site
    pieces (tests/golden/make_golden_large.py sitef)."""
    gam = 2.0 * math.pi / (3.0 * box ** 3)
    full = cfg["intra_site_images"] == "full"
    out = []
    for (idx, forms), lams in zip(sites, lam_values):
        w = weights(lams)
        sp = np.asarray(positions, np.float64)[idx]
        qt = w @ forms
        # Delta E = sum_st W_st (K + G)_st + eta gamma sum_rho w_rho |D_rho|^2
        wm = 0.5 * (np.einsum("r,rs,rt->st", w, forms, forms) - np.outer(qt, qt))
        g = np.zeros_like(sp)
        disp = sp[:, None, :] - sp[None, :, :]
        if full:
            for nvec in image_vectors(0, 1):
                d = disp + nvec * box
                r = np.sqrt((d * d).sum(-1))
                if not nvec.any():
                    np.fill_diagonal(r, np.inf)
                g += 2.0 * np.einsum("it,itx->ix", wm, -d / r[..., None] ** 3)
        else:
            d = disp - box * np.round(disp / box)
            r = np.sqrt((d * d).sum(-1))
            np.fill_diagonal(r, np.inf)
            g += 2.0 * np.einsum("it,itx->ix", wm, -d / r[..., None] ** 3)
        if full and lat is not None:
            rv = regular(sp - 0.5 * box, cfg["p"])
            dr = regular_grad(sp - 0.5 * box, cfg["p"])
            # d/dr_i sum_st W_st Re(R_s T R_t): both slots
            v1 = lat @ (rv.T @ wm.T)  # (nc, ns): column i = T sum_t W_it R_t
            v2 = (wm.T @ rv) @ lat    # (ns, nc): row i = sum_s W_si R_s T
            g += np.real(np.einsum("inx,ni->ix", dr, v1))
            g += np.real(np.einsum("imx,im->ix", dr, v2))
        if full and cfg["dipole"]:
            dev = qt[None, :] - forms
            dd = dev @ (sp - 0.5 * box)
            g += 2.0 * DIPOLE_ETA * gam * np.einsum("r,ri,rx->ix", w, dev, dd)
        out.append(-g)
    return np.concatenate(out) if out else np.zeros((0, 3))


# ------------------------------------------------------ direct sums ----
def direct_potentials(positions, charges, box, shell_cap=0):
    """Brute-force image sum |n|_inf <= shell_cap (oracle.py:33-51)."""
    pos = np.asarray(positions, np.float64)
    q = np.asarray(charges, np.float64)
    disp = pos[:, None, :] - pos[None, :, :]
    v = np.zeros(pos.shape[0])
    for nvec in image_vectors(0, shell_cap):
        d = disp + nvec * box
        r = np.sqrt((d * d).sum(-1))
        if not nvec.any():
            np.fill_diagonal(r, np.inf)
        v += (1.0 / r) @ q
    return v


# ------------------------------------------------------- full CPU step ----
if _nb is not None:
    _p2p_serial = _nb.njit(parallel=False, cache=False)(_p2p_numba.py_func)
else:  # pragma: no cover
    _p2p_serial = None


def full_step(positions, charges, box, sites, lam_values, cfg, clock, serial_near=True):
    """One complete electrostatics step on the host, nothing sampled or
    extrapolated (SURVEY.md §8d step definition): tree + scale_charges
    (system.py:179-197) + solve with near/far/dipole potentials, energies and
    spatial forces in one pass (solver.py:349-427) + HI corrections and
    lambda forces (corrections.py:157-274) + the HI site-atom forces.  The
    near field runs the reference's serial numba loop (solver.py:164-195:
    @njit without parallel) when serial_near; numpy / BLAS use every thread
    they are given (the reference's LAMBDAFMM_THREADS knob, cli.py:35-47).
    Returns (seconds, parts, results)."""
    parts = {}
    t0 = clock()
    q = np.array(charges, np.float64, copy=True)
    for (idx, forms), lams in zip(sites, lam_values):
        q[idx] = weights(lams) @ forms
    pos = wrap(np.atleast_2d(positions), box)
    tree = build_tree(pos, box, cfg["depth"])
    qs = q[tree["perm"]][:, None]
    parts["tree+scale"] = clock() - t0
    t0 = clock()
    if serial_near and _p2p_serial is not None:
        nleaf = tree["leaf_start"].size - 1
        vn = np.zeros((pos.shape[0], 1))
        gn = np.zeros((pos.shape[0], 3))
        rows = np.arange(27) if cfg["periodic_near"] else np.array([13])
        _p2p_serial(tree["positions"], tree["leaf_start"], tree["nb_box"],
                    (tree["nb_shift"] * box).astype(np.float64), np.ascontiguousarray(qs), rows,
                    np.arange(nleaf), True, vn, gn)
    else:
        vn, gn = near_field(tree, qs, cfg["periodic_near"], grad=True)
    parts["p2p"] = clock() - t0
    t0 = clock()
    mult = upward(tree, qs, cfg["p"])
    parts["p2m+m2m"] = clock() - t0
    t0 = clock()
    lat = lattice_matrix(cfg, box)
    root_local = None if lat is None else lat @ mult[0][:, 0, :]
    loc = downward(tree, mult, cfg["p"], root_local)
    parts["lattice+m2l+l2l"] = clock() - t0
    t0 = clock()
    vf, gf = evaluate(tree, loc, cfg["p"], grad=True)
    parts["l2p"] = clock() - t0
    t0 = clock()
    disp = tree["positions"] - 0.5 * box
    dvec = disp.T @ qs
    gam = 2.0 * math.pi / (3.0 * box ** 3)
    if cfg["dipole"]:
        vd = 2.0 * DIPOLE_ETA * gam * (disp @ dvec)
        ed = float(DIPOLE_ETA * gam * (dvec * dvec).sum())
    else:
        vd, ed = np.zeros_like(vn), 0.0
    en = 0.5 * math.fsum((qs[:, 0] * vn[:, 0]).tolist())
    ef = 0.5 * math.fsum((qs[:, 0] * vf[:, 0]).tolist())
    inv = tree["inv_perm"]
    pot = (vn + vf + vd)[inv, 0]
    f = -qs[:, :1] * (gn + gf)
    if cfg["dipole"]:
        f += -2.0 * DIPOLE_ETA * gam * qs[:, :1] * dvec[None, :, 0]
    forces = f[inv]
    res = dict(potentials=pot, energy=en + ef + ed, lattice=lat)
    out = hi(positions, charges, box, sites, lam_values, cfg, solve_out=res)
    if sites:
        idx = np.concatenate([s[0] for s in sites])
        forces[idx] += hi_site_forces(positions, box, sites, lam_values, cfg, lat)
    parts["finalize+hi"] = clock() - t0
    out["spatial_forces"] = forces
    return sum(parts.values()), parts, out


# --------------------------------------------------- timed CPU sample ----
def timed_step_sample(positions, charges, box, sites, lam_values, cfg, fraction, clock):
    """Time one full step (tree + scale + solve + forces + HI) on a bounded
    sample and extrapolate to the whole system.

    Whole-system stages (tree + lists + charge scaling, M2L operator tables,
    lattice, HI) run in full.  Per-target stages (P2P, P2M, M2L+L2L, L2P) run
    on the first `fraction` and `2*fraction` of leaves / boxes; the two
    timings fix a linear model t(f) = a + b f whose value at f = 1 is the
    extrapolated stage time (the intercept keeps per-call overheads from
    being scaled up).  Returns (seconds per step, parts)."""
    parts = {}
    t0 = clock()
    pos = wrap(np.atleast_2d(positions), box)
    tree = build_tree(pos, box, cfg["depth"])
    pairs = {l: m2l_pairs(l) for l in range(1, cfg["depth"] + 1)}  # lists are part of build_octree
    q = np.array(charges, np.float64, copy=True)
    for (idx, forms), lams in zip(sites, lam_values):
        q[idx] = weights(lams) @ forms
    parts["tree+scale"] = clock() - t0
    qs = q[tree["perm"]][:, None]
    nleaf = 8 ** cfg["depth"]
    t0 = clock()
    ops = {l: m2l_level_ops(cfg["p"], box / 2 ** l) for l in range(1, cfg["depth"] + 1)}
    lat = lattice_matrix(cfg, box)
    parts["m2l operators+lattice"] = clock() - t0

    def fit(run):
        ts = []
        fs = []
        for f in (fraction, 2 * fraction):
            f = min(1.0, f)
            t0 = clock()
            run(f)
            ts.append(clock() - t0)
            fs.append(f)
        if fs[1] == fs[0]:
            return ts[1]
        b = max(0.0, (ts[1] - ts[0]) / (fs[1] - fs[0]))
        a = max(0.0, ts[0] - b * fs[0])
        return a + b

    def leaves_of(f):
        return np.arange(max(1, int(math.ceil(f * nleaf))))

    state = {}
    parts["p2p"] = fit(lambda f: near_field(tree, qs, cfg["periodic_near"], grad=True, leaves=leaves_of(f)))

    def up(f):
        state["mult"] = upward(tree, qs, cfg["p"], leaves=leaves_of(f))

    parts["p2m+m2m"] = fit(up)

    def down(f):
        mult = state["mult"]
        root_local = None if lat is None else lat @ mult[0][:, 0, :]
        state["loc"] = downward(tree, mult, cfg["p"], root_local, boxes_fraction=f, ops=ops, pairs=pairs)

    parts["m2l+l2l"] = fit(down)
    parts["l2p"] = fit(lambda f: evaluate(tree, state["loc"], cfg["p"], grad=True, leaves=leaves_of(f)))
    t0 = clock()
    res = dict(potentials=np.zeros(pos.shape[0]), energy=0.0, lattice=lat)
    hi(positions, charges, box, sites, lam_values, cfg, solve_out=res)
    parts["hi"] = clock() - t0
    return sum(parts.values()), parts
