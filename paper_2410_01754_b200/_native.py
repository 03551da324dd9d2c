"""ctypes binding of the in-tree C-ABI library ``_lib/liblfmm.so`` (include/lfmm.h).

This module is the only place Python touches native code.  There is no
fallback: if the library is missing or no CUDA device is present, every
call raises.  Host numpy arrays are passed as plain pointers; device
buffers (torch CUDA tensors) are passed as integer addresses with
``io_on_device=1``.
"""

import ctypes
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("LFMM_LIB") or os.path.join(_HERE, "_lib", "liblfmm.so")

LFMM_LATTICE = {"off": 0, "converged": 1, "shells": 2}
F_DIPOLE, F_PERIODIC_NEAR, F_FP32, F_INTRA_MINIMUM = 1, 2, 4, 8
MODE_HI, MODE_QI = 0, 1


class NumericalFailure(RuntimeError):
    """Non-finite result (the reference CLI's NumericalFailure, cli.py:24-25)."""


class NativeLibraryMissing(RuntimeError):
    pass


_lib = None

_c = ctypes
_vp = _c.c_void_p
_i64 = _c.c_int64
_i32 = _c.c_int
_dbl = _c.c_double


def _declare(lib):
    sig = {
        "lfmm_version": (_c.c_char_p, []),
        "lfmm_last_error": (_i32, [_c.c_char_p, _i64]),
        "lfmm_plan_create": (_i32, [_vp, _i64, _dbl, _i32, _i32, _i32, _i32, _i32, _c.POINTER(_vp)]),
        "lfmm_plan_destroy": (_i32, [_vp]),
        "lfmm_plan_set_stream": (_i32, [_vp, _vp]),
        "lfmm_plan_set_positions": (_i32, [_vp, _vp, _i32]),
        "lfmm_plan_info": (_i32, [_vp, _vp]),
        "lfmm_export_tree": (_i32, [_vp, _vp, _vp, _vp, _vp, _vp]),
        "lfmm_export_lists": (_i32, [_vp, _i32, _vp, _vp, _vp, _vp]),
        "lfmm_lattice_matrix": (_i32, [_vp, _vp]),
        "lfmm_solve": (_i32, [_vp, _vp, _i64, _i32, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp]),
        "lfmm_sites_set": (_i32, [_vp, _i64, _vp, _vp, _vp, _vp, _vp]),
        "lfmm_hi": (_i32, [_vp, _vp, _vp, _i32, _vp, _vp, _i32, _vp, _vp, _vp, _vp, _vp, _vp]),
        "lfmm_assemble": (_i32, [_i64, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _i64, _vp]),
        "lfmm_scale_charges": (_i32, [_vp, _vp, _vp, _vp, _i32, _vp]),
        "lfmm_step": (_i32, [_vp, _vp, _vp, _vp, _vp, _i32, _i32, _i32, _vp, _vp, _vp, _vp]),
        "lfmm_profile_enable": (_i32, [_vp, _i32]),
        "lfmm_stage_count": (_i32, []),
        "lfmm_stage_name": (_c.c_char_p, [_i32]),
        "lfmm_stage_times": (_i32, [_vp, _vp, _vp, _i32]),
        "lfmm_launch_count": (_i64, [_vp]),
        "lfmm_plan_set_count": (_i32, [_vp, _i64]),
        "lfmm_dist_configure": (_i32, [_vp, _i32, _i32, _i32]),
        "lfmm_dist_phase": (_i32, [_vp, _i32, _vp, _vp, _vp, _vp, _i32]),
        "lfmm_dist_buffers": (_i32, [_vp, _vp, _vp, _vp]),
        "lfmm_dist_hi": (_i32, [_vp, _vp, _i32]),
        "lfmm_site_gram": (_i32, [_vp, _vp, _vp, _vp, _vp]),
        "lfmm_hi_site_forces": (_i32, [_vp, _i32, _vp]),
        "lfmm_lambda_baoab": (_i32, [_vp, _i64, _vp, _vp, _vp, _vp, _vp, _vp, _i32, _dbl, _dbl, _dbl, _dbl, _dbl,
                                     _c.c_uint64, _c.c_uint64]),
        "lfmm_lambda_record": (_i32, [_vp, _i64, _vp, _vp, _vp, _vp, _vp, _vp, _dbl, _i64, _vp, _vp, _vp, _vp,
                                      _i64]),
    }
    for name, (res, args) in sig.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args


def exported_symbols():
    """Names declared in include/lfmm.h that the library must export."""
    return [
        "lfmm_version", "lfmm_last_error", "lfmm_plan_create", "lfmm_plan_destroy",
        "lfmm_plan_set_stream", "lfmm_plan_set_positions", "lfmm_plan_info", "lfmm_export_tree",
        "lfmm_export_lists", "lfmm_lattice_matrix", "lfmm_solve", "lfmm_sites_set", "lfmm_hi",
        "lfmm_assemble", "lfmm_scale_charges", "lfmm_step", "lfmm_profile_enable",
        "lfmm_stage_count", "lfmm_stage_name", "lfmm_stage_times", "lfmm_launch_count",
        "lfmm_plan_set_count", "lfmm_dist_configure", "lfmm_dist_phase", "lfmm_dist_buffers", "lfmm_dist_hi",
        "lfmm_site_gram", "lfmm_lambda_baoab", "lfmm_lambda_record", "lfmm_hi_site_forces",
    ]


def lib():
    """Load (once) and return the native library; raises if it is absent."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise NativeLibraryMissing(
                f"{LIB_PATH} not built; run `python -c 'import __graft_entry__ as g; g.build()'` (or `make`)"
            )
        l = ctypes.CDLL(LIB_PATH)
        _declare(l)
        _lib = l
    return _lib


def _err(rc):
    buf = ctypes.create_string_buffer(1024)
    lib().lfmm_last_error(buf, 1024)
    msg = buf.value.decode("utf-8", "replace")
    if rc == 1:
        return ValueError(msg)
    if rc == 3:
        return NumericalFailure(msg)
    return RuntimeError(f"lfmm CUDA failure: {msg}")


def check(rc):
    if rc != 0:
        raise _err(rc)


def ptr(a):
    """Address of a numpy array, a torch tensor, an int, or None."""
    if a is None:
        return None
    if isinstance(a, int):
        return a
    if isinstance(a, np.ndarray):
        return a.ctypes.data
    dp = getattr(a, "data_ptr", None)
    if dp is not None:
        return dp()
    raise TypeError(f"cannot take the address of {type(a)!r}")


def f64(a, shape=None):
    out = np.ascontiguousarray(np.asarray(a, dtype=np.float64))
    if shape is not None:
        out = out.reshape(shape)
    return out


class Plan:
    """Owning handle of one lfmm_plan (one PeriodicSolver's device state)."""

    def __init__(self, positions, box_length, p, depth, lattice_mode, shell_cap, flags):
        pos = f64(positions)
        if pos.ndim != 2 or pos.shape[1] != 3:
            raise ValueError(f"positions must have shape (N, 3), got {pos.shape}")
        self.n = pos.shape[0]
        self.p = int(p)
        self.depth = int(depth)
        self.flags = int(flags)
        self.box_length = float(box_length)
        h = ctypes.c_void_p()
        check(lib().lfmm_plan_create(ptr(pos), self.n, self.box_length, self.p, self.depth,
                                     int(lattice_mode), int(shell_cap), self.flags, ctypes.byref(h)))
        self.h = h
        self.sites_key = None

    def close(self):
        if getattr(self, "h", None) is not None and self.h.value:
            if _lib is not None:
                _lib.lfmm_plan_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @property
    def nc(self):
        return (self.p + 1) ** 2

    def set_stream(self, stream_ptr):
        check(lib().lfmm_plan_set_stream(self.h, stream_ptr))

    def set_positions(self, positions, on_device=False):
        if on_device:
            check(lib().lfmm_plan_set_positions(self.h, ptr(positions), 1))
        else:
            pos = f64(positions, (self.n, 3))
            check(lib().lfmm_plan_set_positions(self.h, ptr(pos), 0))

    def export_tree(self):
        n, nl = self.n, 8 ** self.depth
        perm = np.empty(n, np.int64)
        inv = np.empty(n, np.int64)
        leaf = np.empty(n, np.int64)
        start = np.empty(nl + 1, np.int64)
        pos = np.empty((n, 3), np.float64)
        check(lib().lfmm_export_tree(self.h, ptr(perm), ptr(inv), ptr(leaf), ptr(start), ptr(pos)))
        return perm, inv, leaf, start, pos

    def export_lists(self, level):
        nl = 8 ** self.depth
        nb = np.empty((nl, 27), np.int64)
        sh = np.empty((nl, 27, 3), np.int64)
        if level >= 1:
            nbox = 8 ** level
            src = np.empty((nbox, 189), np.int64)
            row = np.empty((nbox, 189), np.int64)
        else:
            src = row = None
        check(lib().lfmm_export_lists(self.h, int(level), ptr(nb), ptr(sh), ptr(src), ptr(row)))
        return nb, sh, src, row

    def lattice_matrix(self):
        out = np.empty((self.nc, self.nc), np.complex128)
        check(lib().lfmm_lattice_matrix(self.h, ptr(out)))
        return out

    def solve(self, charges, forces=False):
        q = f64(charges)
        k = q.shape[1]
        n = self.n
        pot = np.empty((n, k))
        near = np.empty((n, k))
        far = np.empty((n, k))
        dip = np.empty((n, k))
        en = np.empty((4, k))
        root = np.empty((self.nc, k), np.complex128)
        dvec = np.empty((3, k))
        qtot = np.empty(k)
        frc = np.empty((n, 3)) if forces else None
        check(lib().lfmm_solve(self.h, ptr(q), k, 0, ptr(pot), ptr(near), ptr(far), ptr(dip), ptr(en),
                               ptr(root), ptr(dvec), ptr(qtot), ptr(frc)))
        return dict(potentials=pot, near=near, far=far, dip=dip, energies=en, root=root, dipole=dvec,
                    qtot=qtot, forces=frc)

    def set_sites(self, atom_offsets, atom_index, n_forms, form_offsets, form_charges, key=None):
        ao = np.ascontiguousarray(atom_offsets, dtype=np.int64)
        ai = np.ascontiguousarray(atom_index, dtype=np.int64)
        nf = np.ascontiguousarray(n_forms, dtype=np.int32)
        fo = np.ascontiguousarray(form_offsets, dtype=np.int64)
        fq = np.ascontiguousarray(form_charges, dtype=np.float64)
        check(lib().lfmm_sites_set(self.h, len(nf), ptr(ao), ptr(ai), ptr(nf), ptr(fo), ptr(fq)))
        self.sites_key = key
        self.n_sites = len(nf)
        self.n_site_atoms = int(ao[-1]) if len(ao) else 0
        self.n_form_slots = int(nf.sum())
        self.form_slot_offsets = np.concatenate([[0], np.cumsum(nf)]).astype(np.int64)

    def hi(self, lambdas, n_lambda, mode, site_positions=None, potentials=None, want_forces=True):
        s = self.n_sites
        lam = f64(lambdas, (s, 4)) if s else np.zeros((0, 4))
        nl = np.ascontiguousarray(n_lambda, dtype=np.int32)
        sp = None if site_positions is None else f64(site_positions)
        pot = None if potentials is None else f64(potentials)
        f = self.n_form_slots
        cp, cl, cd = np.empty(f), np.empty(f), np.empty(f)
        eb = np.empty(s)
        lf = np.empty((s, 4)) if want_forces else None
        off = np.empty(1)
        check(lib().lfmm_hi(self.h, ptr(lam), ptr(nl), int(mode), ptr(sp), ptr(pot), 0, ptr(cp), ptr(cl),
                            ptr(cd), ptr(eb), ptr(lf), ptr(off)))
        return dict(c_p2p=cp, c_lattice=cl, c_dipole=cd, blend=eb, forces=lf, offset=float(off[0]))

    def hi_site_forces(self):
        """(A, 3) -grad Delta E_site of the last HI-mode correction pass."""
        out = np.empty((self.n_site_atoms, 3))
        check(lib().lfmm_hi_site_forces(self.h, 0, ptr(out)))
        return out

    def scale_charges(self, charges, lambdas, n_lambda):
        q = f64(charges, (self.n,))
        out = np.empty(self.n)
        lam = f64(lambdas, (self.n_sites, 4))
        nl = np.ascontiguousarray(n_lambda, dtype=np.int32)
        check(lib().lfmm_scale_charges(self.h, ptr(q), ptr(lam), ptr(nl), 0, ptr(out)))
        return out

    def step(self, positions, charges, lambdas, n_lambda, mode=MODE_HI, plain=False, on_device=False,
             energy=None, forces=None, lambda_forces=None, potentials=None):
        check(lib().lfmm_step(self.h, ptr(positions), ptr(charges), ptr(lambdas), ptr(n_lambda), int(mode),
                              1 if plain else 0, 1 if on_device else 0, ptr(energy), ptr(forces),
                              ptr(lambda_forces), ptr(potentials)))

    def profile(self, enable):
        check(lib().lfmm_profile_enable(self.h, 1 if enable else 0))

    def stage_times(self):
        n = lib().lfmm_stage_count()
        ms = np.zeros(n)
        cnt = np.zeros(n, np.int64)
        check(lib().lfmm_stage_times(self.h, ptr(ms), ptr(cnt), n))
        names = [lib().lfmm_stage_name(i).decode() for i in range(n)]
        return {nm: (float(m), int(c)) for nm, m, c in zip(names, ms, cnt)}

    def launch_count(self):
        return int(lib().lfmm_launch_count(self.h))

    # ---- lambda dynamics (dynamics.py) ----
    def site_gram(self, lambdas, n_lambda, site_positions):
        """(S, 16, 16) per-site Q (K + G) Q^T."""
        out = np.zeros((self.n_sites, 16, 16))
        check(lib().lfmm_site_gram(self.h, ptr(lambdas), ptr(n_lambda), ptr(site_positions), ptr(out)))
        return out

    def lambda_baoab(self, n_sites, lam, vel, n_lambda, masses, f_engine, f_total, stage, dt, coulomb, bias_height,
                     c1, noise, seed, step):
        check(lib().lfmm_lambda_baoab(self.h, int(n_sites), ptr(lam), ptr(vel), ptr(n_lambda), ptr(masses),
                                      ptr(f_engine), ptr(f_total), int(stage), float(dt), float(coulomb),
                                      float(bias_height), float(c1), float(noise), int(seed), int(step)))

    def lambda_record(self, n_sites, slot_off, n_lambda, lam, vel, f_total, energy, coulomb, n_slots, out_x, out_v,
                      out_f, out_e, sample):
        check(lib().lfmm_lambda_record(self.h, int(n_sites), ptr(slot_off), ptr(n_lambda), ptr(lam), ptr(vel),
                                       ptr(f_total), ptr(energy), float(coulomb), int(n_slots), ptr(out_x),
                                       ptr(out_v), ptr(out_f), ptr(out_e), int(sample)))

    # ---- slab decomposition (distributed.py) ----
    def set_count(self, n):
        check(lib().lfmm_plan_set_count(self.h, int(n)))
        self.n = int(n)

    def dist_configure(self, x0, x1, lg):
        check(lib().lfmm_dist_configure(self.h, int(x0), int(x1), int(lg)))

    def dist_phase(self, phase, positions=None, charges=None, lambdas=None, n_lambda=None, grad=True):
        check(lib().lfmm_dist_phase(self.h, int(phase), ptr(positions), ptr(charges), ptr(lambdas), ptr(n_lambda),
                                    1 if grad else 0))

    def dist_buffers(self):
        ptrs = (ctypes.c_void_p * 9)()
        offs = np.zeros(8, np.int64)
        ncp = np.zeros(1, np.int64)
        check(lib().lfmm_dist_buffers(self.h, ptrs, ptr(offs), ptr(ncp)))
        self.ncp = int(ncp[0])
        return [p if p is not None else 0 for p in ptrs], offs

    def dist_hi(self, site_positions, mode=MODE_HI):
        check(lib().lfmm_dist_hi(self.h, ptr(site_positions), int(mode)))


def assemble(atom_offsets, atom_index, n_forms, form_offsets, form_charges, lambdas, n_lambda, c_total,
             potentials):
    """Device lambda-force assembly without a plan (assemble_lambda_forces)."""
    ao = np.ascontiguousarray(atom_offsets, dtype=np.int64)
    ai = np.ascontiguousarray(atom_index, dtype=np.int64)
    nf = np.ascontiguousarray(n_forms, dtype=np.int32)
    fo = np.ascontiguousarray(form_offsets, dtype=np.int64)
    fq = np.ascontiguousarray(form_charges, dtype=np.float64)
    s = len(nf)
    lam = f64(lambdas, (s, 4))
    nl = np.ascontiguousarray(n_lambda, dtype=np.int32)
    ct = None if c_total is None else f64(c_total)
    pot = f64(potentials).reshape(-1)
    out = np.empty((s, 4))
    check(lib().lfmm_assemble(s, ptr(ao), ptr(ai), ptr(nf), ptr(fo), ptr(fq), ptr(lam), ptr(nl), ptr(ct),
                              ptr(pot), pot.shape[0], ptr(out)))
    return out
