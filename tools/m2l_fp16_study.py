"""Design study (not product code): accuracy of a fp16x3 tensor-core M2L.

Builds the 316 box-normalised M2L operators in the packed real layout the
device uses, equilibrates them with power-of-two row/column scales, and
compares the level-d M2L of a synthetic water box (oracle multipoles, fp64)
computed exactly against emulated operand roundings:

  fp32      : operands rounded to fp32 (the SIMT kernel)
  tf32x3    : a ~ hi + lo in tf32, products hi*hi + hi*lo + lo*hi
  fp16x3    : same with fp16 hi/lo after scaling (subnormals kept)
  fp16x1    : one fp16 product (for scale)

  far2b     : fp16x3, but two products (operator hi only) on the outer-shell
              offsets (|o|inf = 3: 218 of the 316 operators)

Error metric: max |dV| / max |V| of the potential the level-d locals produce
at the particles (L2P), i.e. the reference's max-normalised metric applied to
this stage's contribution alone (stricter than on the total far potential).
"""

import sys

import numpy as np

sys.path.insert(0, ".")
from oracle import lfmm_oracle as orc  # noqa: E402


def pk_list(p):
    out = []
    for l in range(p + 1):
        out.append((l, 0, 0))
    for m in range(1, p + 1):
        for l in range(m, p + 1):
            out.append((l, m, 0))
            out.append((l, m, 1))
    return out


def to_complex_basis(p):
    """(nc_complex, npk) matrix E with full complex coeffs = E @ packed."""
    pk = pk_list(p)
    nc = orc.ncoef(p)
    E = np.zeros((nc, len(pk)), np.complex128)
    for b, (l, m, part) in enumerate(pk):
        v = 1.0 if part == 0 else 1.0j
        E[orc.cidx(l, m), b] += v
        if m > 0:
            E[orc.cidx(l, -m), b] += (-1) ** m * np.conj(v)
    return E


def from_complex(p):
    """(npk, nc) real extraction: packed = Re/Im of the m >= 0 entries."""
    pk = pk_list(p)
    nc = orc.ncoef(p)
    P = np.zeros((len(pk), nc), np.complex128)
    for a, (l, m, part) in enumerate(pk):
        # Re z = (z)_re ; we build with complex and take real parts after
        P[a, orc.cidx(l, m)] = 1.0 if part == 0 else -1.0j
    return P


def real_ops(p):
    E = to_complex_basis(p)
    P = from_complex(p)
    iv = orc.irregular(orc.M2L_OFF.astype(float), 2 * p)
    ops = []
    for row in range(orc.M2L_OFF.shape[0]):
        B = orc.m2l_from_iv(iv[row], p)
        ops.append(np.real(P @ B @ E))
    return np.array(ops)  # (316, npk, npk)


def pow2(x):
    return 2.0 ** np.round(np.log2(x))


def equilibrate(ops, iters=30):
    n = ops.shape[1]
    r = np.ones(n)
    c = np.ones(n)
    A = np.abs(ops).max(0)
    for _ in range(iters):
        S = r[:, None] * A * c[None, :]
        r = r / np.sqrt(S.max(1))
        S = r[:, None] * A * c[None, :]
        c = c / np.sqrt(S.max(0))
    return pow2(r), pow2(c)


def tf32(x):
    x = np.asarray(x, np.float32)
    u = x.view(np.uint32).astype(np.uint64)
    u = ((u + 0x1000) & 0xFFFFE000).astype(np.uint32)
    return u.view(np.float32).astype(np.float64)


def split(x, kind):
    if kind == "tf32":
        hi = tf32(x)
        lo = tf32(np.float32(x - hi))
    else:
        hi = np.asarray(x, np.float16).astype(np.float64)
        lo = np.asarray(x - hi, np.float16).astype(np.float64)
    return hi, lo


def main():
    p = 10
    n_atoms = int(sys.argv[1]) if len(sys.argv) > 1 else 100000
    depth = int(sys.argv[2]) if len(sys.argv) > 2 else 4
    from paper_2410_01754_b200.waterbox import generate_water_box

    system, lam, _ = generate_water_box(n_atoms, 8, seed=0)
    pos, q, box = system.positions, system.charges, system.box_length
    tree = orc.build_tree(orc.wrap(pos, box), box, depth)
    qs = q[tree["perm"]][:, None]
    mult = orc.upward(tree, qs, p)
    ops = real_ops(p)
    r, c = equilibrate(ops)
    Bs = r[None, :, None] * ops * c[None, None, :]
    print("operator entries after scaling: max %.3g, min nonzero %.3g" % (np.abs(Bs).max(), np.abs(Bs[Bs != 0]).min()))
    P = from_complex(p)
    E = to_complex_basis(p)
    pk = pk_list(p)
    lvec = np.array([l for (l, m, part) in pk])
    results = {}
    for level in (depth,):
        n = 2 ** level
        size = box / n
        M = np.real(P @ mult[level][:, :, 0])  # (npk, nbox)
        Mh = M / size ** lvec[:, None]  # normalised
        Ms = Mh / c[:, None]
        print("level %d: max|M^| %.3g  max|M^/c| %.3g  min|M^/c|>0 %.3g" %
              (level, np.abs(Mh).max(), np.abs(Ms).max(), np.abs(Ms[Ms != 0]).min()))
        gl = 2.0 ** (12 - np.ceil(np.log2(np.abs(Ms).max())))
        pairs = orc.m2l_pairs(level)
        variants = {"exact": None, "fp32": None, "tf32x3": None, "fp16x3": None, "fp16x2a": None,
                    "fp16x2b": None, "fp16x1": None, "far2b": None}
        if len(sys.argv) > 3:
            variants = {k: None for k in sys.argv[3].split(",")}
        far = np.abs(orc.M2L_OFF).max(1) >= 3  # outer shell of the interaction list
        r2min = float(sys.argv[4]) if len(sys.argv) > 4 else 0.0
        if r2min > 0:  # far2b on the offsets with |o|^2 >= r2min only
            far = (orc.M2L_OFF ** 2).sum(1) >= r2min
        print("far2b offsets: %d of %d" % (far.sum(), len(far)))
        locs = {}
        for name in variants:
            Lh = np.zeros_like(Mh)
            for row, t, s in pairs:
                if name == "exact":
                    Lh[:, t] += ops[row] @ Mh[:, s]
                elif name == "fp32":
                    Lh[:, t] += ops[row].astype(np.float32).astype(np.float64) @ Mh[:, s].astype(np.float32).astype(np.float64)
                elif name == "tf32x3":
                    ah, al = split(ops[row], "tf32")
                    bh, bl = split(Mh[:, s], "tf32")
                    Lh[:, t] += ah @ bh + ah @ bl + al @ bh
                elif name == "fp16x3":
                    ah, al = split(Bs[row], "fp16")
                    bh, bl = split(Ms[:, s] * gl, "fp16")
                    Lh[:, t] += ((ah @ bh + ah @ bl + al @ bh) / r[:, None]) / gl
                elif name == "fp16x2a":  # operator hi/lo, multipoles one fp16
                    ah, al = split(Bs[row], "fp16")
                    bh = np.asarray(Ms[:, s] * gl, np.float16).astype(np.float64)
                    Lh[:, t] += ((ah @ bh + al @ bh) / r[:, None]) / gl
                elif name == "fp16x2b":  # operator one fp16, multipoles hi/lo
                    ah = np.asarray(Bs[row], np.float16).astype(np.float64)
                    bh, bl = split(Ms[:, s] * gl, "fp16")
                    Lh[:, t] += ((ah @ bh + ah @ bl) / r[:, None]) / gl
                elif name == "far2b":  # operator one fp16 on the outer-shell offsets only
                    ah, al = split(Bs[row], "fp16")
                    bh, bl = split(Ms[:, s] * gl, "fp16")
                    acc = ah @ bh + ah @ bl if far[row] else ah @ bh + ah @ bl + al @ bh
                    Lh[:, t] += (acc / r[:, None]) / gl
                elif name == "fp16x1":
                    ah = np.asarray(Bs[row], np.float16).astype(np.float64)
                    bh = np.asarray(Ms[:, s] * gl, np.float16).astype(np.float64)
                    Lh[:, t] += ((ah @ bh) / r[:, None]) / gl
            locs[name] = Lh
        # L2P of this level's locals at the particles
        cen = orc.leaf_centers(tree) if level == depth else None
        lof = tree["leaf_of_particle"]
        disp = tree["positions"] - cen[lof]
        R = orc.regular(disp / size, p)  # normalised: L^ R(r/s)/s
        Rp = np.real(R @ E)  # packed basis evaluation: V = sum_b Re(R E)_b L_b ... check below
        V = {}
        for name, Lh in locs.items():
            Lc = E @ Lh  # complex full coefficients
            V[name] = np.real(np.einsum("nc,cn->n", R, Lc[:, lof])) / size
        vmax = np.abs(V["exact"]).max()
        for name in locs:
            if name == "exact":
                continue
            err = np.abs(V[name] - V["exact"]).max() / vmax
            lerr = np.abs(locs[name] - locs["exact"]).max() / np.abs(locs["exact"]).max()
            results[name] = err
            print("  %-7s  V err (max-normalised) %.3e   local coeff err %.3e" % (name, err, lerr))
        del Rp
    return results


if __name__ == "__main__":
    main()
