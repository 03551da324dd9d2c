"""Octree slab decomposition of the FMM + HI step over ranks.

One rank per GPU.  Rank r of G (G a power of two, G <= 2^depth) owns the
leaves with x index in [r w, (r+1) w), w = 2^depth / G, i.e. the level-lg
boxes with x index r for lg = log2 G (G = 8: the 8 level-1 octants become x
slabs of the leaf grid; the reference is single-process, so the layout is
ours).  Per step and rank:

1. particle halo exchange with the two neighbour ranks (point-to-point):
   each rank holds its own atoms (global ids) and sends the atoms of its
   boundary leaf planes (the neighbours' P2P halo, solver.py:126-195) and
   those that moved into a neighbour's slab (handed over); `step` starts
   from global arrays and keeps the owned atoms;
2. native phase 1 (lfmm_dist_phase): tree, charges (+ scale_charges), P2P of
   owned leaves, P2M, M2M of levels >= lg (owned subtrees are complete),
   exact box charges, the slab's per-level max |M| (fp16 M2L scales);
3. exchange: level lg all-gathered (it feeds the shared levels); levels > lg
   send/recv only the 2-plane multipole halo each side (the M2L sources of
   the owned targets, octree.py:96-111); per-level max |M| max-reduced; the
   per-rank dipole / charge sums added in rank order;
4. native phase 2: M2M of the shared levels < lg (redundant on every rank),
   lattice, M2L restricted to owned targets (levels >= lg), L2L, L2P of owned
   leaves, finalize (energies of owned atoms), owned site-atom potentials;
5. exchange: energies (near/far partials, rank order), site-atom potentials
   and positions (each atom owned by exactly one rank: exact);
6. HI corrections + lambda forces for all sites (redundant, cheap) from the
   gathered site potentials (corrections.py:157-238).

Every reduction adds per-rank partials in rank order, so results do not
depend on the collective's internal order; multipoles, M2L and P2P of a box
are computed exactly as on one GPU (same jobs restricted to owned targets).

Collectives go through a small `Comm` interface: `TorchComm` wraps a
torch.distributed process group (NCCL for device tensors; gloo stages through
host memory), `LocalComm` simulates G ranks as threads of one process on one
GPU (used by the GPU tests, since the test boxes have one GPU).
"""

import math
import os
import threading

import numpy as np

from . import _native
from .fmm.solver import SolverConfig

_DEBUG = os.environ.get('LFMM_DIST_DEBUG') == '1'
_POISON = os.environ.get('LFMM_DIST_POISON') == '1'
HALO_PLANES = 2  # multipole halo width (x-planes) of the M2L sources at levels > lg

# --------------------------------------------------------------- layout ----


def slab_partition(depth, world):
    """(lg, [(x0, x1) per rank]) for the x-slab decomposition of the leaf grid."""
    n = 1 << depth
    if world < 1 or world & (world - 1):
        raise ValueError(f"world size {world} is not a power of two")
    if world > n:
        raise ValueError(f"world size {world} exceeds the {n} leaf planes of depth {depth}")
    lg = int(round(math.log2(world)))
    w = n // world
    return lg, [(r * w, (r + 1) * w) for r in range(world)]


def leaf_x(positions_wrapped, box_length, depth, xp=np):
    """Leaf x index of wrapped positions, as octree.build_octree assigns it
    (floor(x / size) clipped, octree.py:121-123)."""
    n = 1 << depth
    size = box_length / n
    c = xp.floor(positions_wrapped[:, 0] / size)
    return xp.clip(c, 0, n - 1).astype(xp.int64) if xp is np else c.clamp(0, n - 1).long()


def wrap(positions, box_length, xp=np):
    """np.mod wrap with exact box multiples -> 0 (system.py:103-108)."""
    w = xp.remainder(positions, box_length)
    return xp.where(w >= box_length, xp.zeros_like(w), w)


def select_local(lx, x0, x1, depth, xp=np):
    """Owned atom indices (leaf x in [x0, x1)) and halo indices (leaf planes
    x0-1 and x1, periodic, not owned), each in global input order."""
    n = 1 << depth
    owned = (lx >= x0) & (lx < x1)
    hx = {(x0 - 1) % n, x1 % n}
    halo = xp.zeros_like(owned)
    for h in hx:
        halo = halo | (lx == h)
    halo = halo & ~owned
    if xp is np:
        return np.flatnonzero(owned), np.flatnonzero(halo)
    return owned.nonzero().flatten(), halo.nonzero().flatten()


# ------------------------------------------------------------ collectives ----


def _halo_ops(rank, world, x0, x1, n, width=2):
    """The point-to-point operations of one rank's halo-plane exchange, as
    (kind, peer, first plane).  The owned slab [x0, x1) of n periodic planes
    needs planes x0-width .. x0-1 (the left neighbour's last planes) and
    x1 .. x1+width-1 (the right neighbour's first planes).  Per peer the
    sends and receives are listed in matching order: a rank sends its last
    planes before its first, and receives its left halo before its right
    (with 2 ranks both neighbours are the same peer)."""
    if x1 - x0 < width:
        raise ValueError(f"slab of {x1 - x0} planes is thinner than the halo width {width}")
    left, right = (rank - 1) % world, (rank + 1) % world
    return [("send", right, x1 - width), ("send", left, x0),
            ("recv", left, (x0 - width) % n), ("recv", right, x1 % n)]


def halo_planes(x0, x1, n, width=2):
    """Plane indices a slab's halo exchange fills (periodic)."""
    return sorted({(x0 - k) % n for k in range(1, width + 1)} | {(x1 + k) % n for k in range(width)})


def torch_empty_like_cpu(t):
    import torch

    return torch.empty(t.shape, dtype=t.dtype)



class TorchComm:
    """torch.distributed group; deterministic sums (all-gather + rank order)."""

    def __init__(self, group=None):
        import torch.distributed as dist

        self.dist = dist
        self.group = group
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)
        self.backend = dist.get_backend(group)

    def _staged(self, t):
        return self.backend == "gloo" and t.is_cuda

    def allgather_(self, out, chunk_numel):
        """In place: out (world * chunk) holds this rank's chunk at rank*chunk."""
        mine = out[self.rank * chunk_numel:(self.rank + 1) * chunk_numel].clone()
        if self._staged(out):
            host = out.cpu()
            self.dist.all_gather_into_tensor(host, mine.cpu(), group=self.group)
            out.copy_(host)
        else:
            self.dist.all_gather_into_tensor(out, mine, group=self.group)

    def halo_(self, out, plane_numel, x0, x1, n, width=2):
        """In place: out holds the n x-planes of one level (plane_numel
        elements each), this rank's planes [x0, x1) filled.  Receives the
        `width` planes either side of the slab (periodic) from the neighbour
        ranks, which own them, and sends this rank's first / last `width`
        planes to the left / right neighbour.  Requires x1 - x0 >= width."""
        dist = self.dist
        ops = []
        for kind, peer, a in _halo_ops(self.rank, self.world, x0, x1, n, width):
            seg = out[a * plane_numel:(a + width) * plane_numel]
            ops.append((kind, peer, seg))
        if self._staged(out):
            host = [(k, pr, seg.cpu() if k == "send" else torch_empty_like_cpu(seg)) for k, pr, seg in ops]
            reqs = dist.batch_isend_irecv([dist.P2POp(dist.isend if k == "send" else dist.irecv, h, pr, self.group)
                                           for k, pr, h in host])
            for r in reqs:
                r.wait()
            for (k, _, seg), (_, _, h) in zip(ops, host):
                if k == "recv":
                    seg.copy_(h)
        else:
            reqs = dist.batch_isend_irecv([dist.P2POp(dist.isend if k == "send" else dist.irecv, seg, pr, self.group)
                                           for k, pr, seg in ops])
            for r in reqs:
                r.wait()

    def exchange_(self, sends):
        """Variable-size point-to-point exchange: sends = {peer: (m, k)
        tensor}; returns {peer: the (m', k) tensor that peer sent here}.  The
        row counts travel first (one host sync), then the payloads."""
        import torch

        dist = self.dist
        peers = list(sends)
        dev = next(iter(sends.values())).device
        staged = self.backend == "gloo" and dev.type == "cuda"
        cdev = "cpu" if staged else dev
        cnt_out = {p: torch.tensor([sends[p].shape[0]], dtype=torch.int64, device=cdev) for p in peers}
        cnt_in = {p: torch.empty(1, dtype=torch.int64, device=cdev) for p in peers}
        ops = [dist.P2POp(dist.isend, cnt_out[p], p, self.group) for p in peers]
        ops += [dist.P2POp(dist.irecv, cnt_in[p], p, self.group) for p in peers]
        for r in dist.batch_isend_irecv(ops):
            r.wait()
        out = {}
        ops = []
        counts = torch.cat([cnt_in[p] for p in peers]).tolist()  # the one host sync of the exchange
        for p, m in zip(peers, counts):
            t = sends[p]
            src = t.cpu().contiguous() if staged else t.contiguous()
            out[p] = torch.empty((int(m),) + tuple(t.shape[1:]), dtype=t.dtype, device=cdev)
            ops.append(dist.P2POp(dist.isend, src, p, self.group))
            ops.append(dist.P2POp(dist.irecv, out[p], p, self.group))
        for r in dist.batch_isend_irecv(ops):
            r.wait()
        return {p: v.to(dev) for p, v in out.items()} if staged else out

    def max_(self, t):
        """In place: elementwise max of t over ranks (exact in any order)."""
        import torch

        buf = torch.empty((self.world,) + tuple(t.shape), dtype=t.dtype, device=t.device)
        n = t.numel()
        buf.reshape(-1)[self.rank * n:(self.rank + 1) * n].copy_(t.reshape(-1))
        self.allgather_(buf.reshape(-1), n)
        t.copy_(buf.amax(0))

    def sum_ordered(self, t):
        """Sum of every rank's t, added in rank order (bit-reproducible)."""
        import torch

        buf = torch.empty((self.world,) + tuple(t.shape), dtype=t.dtype, device=t.device)
        flat = buf.reshape(-1)
        n = t.numel()
        flat[self.rank * n:(self.rank + 1) * n].copy_(t.reshape(-1))
        self.allgather_(flat, n)
        acc = buf[0].clone()
        for r in range(1, self.world):
            acc += buf[r]
        return acc


class LocalComm:
    """G ranks as threads of one process sharing one GPU (tests)."""

    def __init__(self, world):
        self.world = world
        self.barrier = threading.Barrier(world)
        self.slots = [None] * world

    def for_rank(self, rank):
        return _LocalRankComm(self, rank)


class _LocalRankComm:
    def __init__(self, shared, rank):
        self.shared = shared
        self.rank = rank
        self.world = shared.world

    def allgather_(self, out, chunk_numel):
        import torch

        torch.cuda.current_stream().synchronize()
        self.shared.slots[self.rank] = out[self.rank * chunk_numel:(self.rank + 1) * chunk_numel]
        self.shared.barrier.wait()
        for r in range(self.world):
            if r != self.rank:
                out[r * chunk_numel:(r + 1) * chunk_numel].copy_(self.shared.slots[r])
        torch.cuda.current_stream().synchronize()
        self.shared.barrier.wait()

    def halo_(self, out, plane_numel, x0, x1, n, width=2):
        import torch

        torch.cuda.current_stream().synchronize()
        self.shared.slots[self.rank] = out
        self.shared.barrier.wait()
        for kind, peer, a in _halo_ops(self.rank, self.world, x0, x1, n, width):
            if kind == "recv":
                out[a * plane_numel:(a + width) * plane_numel].copy_(
                    self.shared.slots[peer][a * plane_numel:(a + width) * plane_numel])
        torch.cuda.current_stream().synchronize()
        self.shared.barrier.wait()

    def exchange_(self, sends):
        import torch

        torch.cuda.current_stream().synchronize()
        self.shared.slots[self.rank] = sends
        self.shared.barrier.wait()
        out = {p: self.shared.slots[p][self.rank].clone() for p in sends}
        torch.cuda.current_stream().synchronize()
        self.shared.barrier.wait()
        return out

    def max_(self, t):
        import torch

        torch.cuda.current_stream().synchronize()
        self.shared.slots[self.rank] = t.clone()
        self.shared.barrier.wait()
        acc = self.shared.slots[0].clone()
        for r in range(1, self.world):
            acc = torch.maximum(acc, self.shared.slots[r])
        torch.cuda.current_stream().synchronize()
        self.shared.barrier.wait()
        t.copy_(acc)

    def sum_ordered(self, t):
        import torch

        buf = torch.empty((self.world,) + tuple(t.shape), dtype=t.dtype, device=t.device)
        flat = buf.reshape(-1)
        n = t.numel()
        flat[self.rank * n:(self.rank + 1) * n].copy_(t.reshape(-1))
        self.allgather_(flat, n)
        acc = buf[0].clone()
        for r in range(1, self.world):
            acc += buf[r]
        return acc


# --------------------------------------------------------------- solver ----


def _device_view(address, shape, dtype_str, torch):
    """A torch tensor over native device memory (__cuda_array_interface__)."""

    class _Arr:
        __cuda_array_interface__ = {"shape": tuple(shape), "typestr": dtype_str, "data": (int(address), False),
                                    "version": 3, "strides": None}

    return torch.as_tensor(_Arr(), device="cuda")


class DistributedSolver:
    """One rank of the slab-decomposed FMM + HI step.

    `step_owned` takes this rank's atoms (positions, charges, global ids)
    plus the lambda table and global site tables, exchanges the boundary
    atoms with the neighbour ranks and returns the global energy, the owned
    forces (global ids) and the lambda forces of every site.  `step` takes
    the global arrays on every rank and keeps the owned atoms.
    """

    def __init__(self, box_length, config=None, comm=None, depth=None):
        import torch

        self.torch = torch
        self.cfg = (config or SolverConfig()).validated()
        if self.cfg.depth < 1:
            raise ValueError("the slab decomposition needs depth >= 1")
        self.box = float(box_length)
        self.comm = comm
        self.rank, self.world = comm.rank, comm.world
        self.lg, ranges = slab_partition(self.cfg.depth, self.world)
        self.x0, self.x1 = ranges[self.rank]
        self.plan = None
        self.flags = (_native.F_DIPOLE if self.cfg.dipole else 0) | _native.F_PERIODIC_NEAR | (
            _native.F_FP32 if self.cfg.precision == "single" else 0) | (
            _native.F_INTRA_MINIMUM if self.cfg.intra_site_images == "minimum" else 0)
        self.tsize = 4 if self.cfg.precision == "single" else 8
        self.stream = None
        self._site_dev = self._site_key = self._site_local = None

    def _ensure_plan(self, pos_local_host):
        if self.plan is None:
            self.plan = _native.Plan(pos_local_host, self.box, self.cfg.p, self.cfg.depth,
                                     _native.LFMM_LATTICE[self.cfg.lattice_mode], self.cfg.shell_cap, self.flags)
            # the plan's kernels and torch's copies / collectives share one
            # (non-default) stream, so they are ordered
            self.plan.set_stream(self.stream.cuda_stream)
            self.plan.dist_configure(self.x0, self.x1, self.lg)

    def step(self, positions, charges, lambdas=None, n_lambda=None, sites=None, site_positions=None,
             mode=_native.MODE_HI):
        """Global inputs on every rank: positions (N,3) f64, charges (N,) f64
        on the device (input order); lambdas (S,4) f64 / n_lambda (S,) i32
        device; sites = (atom offsets (S+1), global atom indices (A), n_forms
        (S), form offsets (S+1), form charges) host arrays.  The rank keeps
        its owned atoms and runs `step_owned` (the halo comes from the
        neighbour ranks, not from the global arrays).  site_positions is
        accepted for compatibility and ignored: the site-atom positions are
        gathered from their owners."""
        torch = self.torch
        w = wrap(positions, self.box, xp=torch)
        lx = leaf_x(w, self.box, self.cfg.depth, xp=torch)
        own = ((lx >= self.x0) & (lx < self.x1)).nonzero().flatten()
        return self.step_owned(positions[own], charges[own], own, lambdas, n_lambda, sites,
                               n_global=positions.shape[0], mode=mode)

    def step_owned(self, positions, charges, global_ids, lambdas=None, n_lambda=None, sites=None, n_global=None,
                   mode=_native.MODE_HI):
        """One step from this rank's own atoms: positions (n,3) f64 (raw,
        unwrapped), charges (n,) f64 and global ids (n,) int64 on the device,
        normally the atoms whose leaf x lies in the rank's slab.  Atoms that
        moved into a neighbour's boundary plane (one leaf plane at most) are
        handed over in the halo exchange.  Returns the global energies, the
        lambda forces of every site, and "owned" / "owned_positions" /
        "owned_charges" / "forces" for the atoms this rank owns after the
        exchange (carry them into the next step)."""
        if self.stream is None:
            self.stream = self.torch.cuda.Stream()
        self.stream.wait_stream(self.torch.cuda.current_stream())
        with self.torch.cuda.stream(self.stream):
            out = self._step(positions, charges, global_ids, lambdas, n_lambda, sites, n_global, mode)
        self.torch.cuda.current_stream().wait_stream(self.stream)
        return out

    def _exchange_particles(self, positions, charges, global_ids):
        """Halo particle exchange with the neighbour ranks (SURVEY.md §8e
        exchange 1).  Sends to the left rank the atoms in leaf planes x0 (its
        right halo) and x0-1 (migrated into its slab), to the right rank those
        in x1-1 and x1; keeps the atoms in [x0, x1) and, as halo, the ones
        that migrated out (they lie in planes x0-1 / x1).  Returns (positions,
        charges, global ids) of the owned atoms followed by the halo atoms,
        and the owned count."""
        torch = self.torch
        d = self.cfg.depth
        n = 1 << d
        x0, x1 = self.x0, self.x1
        lx = leaf_x(wrap(positions, self.box, xp=torch), self.box, d, xp=torch)
        stay = (lx >= x0) & (lx < x1)
        if self.world == 1:
            if not bool(stay.all()):
                raise ValueError("atom outside the grid")
            return positions, charges, global_ids, positions.shape[0]
        xl, xr = (x0 - 1) % n, x1 % n
        to_left = (lx == x0) | (lx == xl)
        to_right = (lx == x1 - 1) | (lx == xr)
        # both migration checks and the kept-atom count in one host sync
        far, moved, n_stay = torch.stack([(~(stay | (lx == xl) | (lx == xr))).any().to(torch.int64),
                                          (~stay).any().to(torch.int64), stay.sum()]).tolist()
        if far:
            raise ValueError("an atom moved more than one leaf plane out of its rank's slab; "
                             "re-partition from global positions (DistributedSolver.step)")
        if x1 - x0 < 2 and self.world > 2 and moved:
            # with one plane per rank a migrant into plane x1 (x0-1) is also
            # the halo of rank r+2 (r-2), which this one-hop exchange never
            # reaches: those pairs would silently drop out of the P2P
            raise ValueError("atoms migrated between ranks that own a single leaf plane each; "
                             "re-partition from global positions (DistributedSolver.step) or use a deeper tree")
        rows = torch.cat([positions, charges[:, None], global_ids.to(torch.float64)[:, None]], 1)
        left, right = (self.rank - 1) % self.world, (self.rank + 1) % self.world
        if left == right:
            recv = self.comm.exchange_({left: rows[to_left | to_right]})
            rec = recv[left]
        else:
            recv = self.comm.exchange_({left: rows[to_left], right: rows[to_right]})
            rec = torch.cat([recv[left], recv[right]])
        rlx = leaf_x(wrap(rec[:, :3].contiguous(), self.box, xp=torch), self.box, d, xp=torch)
        r_own = (rlx >= x0) & (rlx < x1)
        r_halo = ~r_own
        gone = ~stay  # migrated to a neighbour's boundary plane: still in this rank's halo
        pos = torch.cat([positions[stay], rec[r_own, :3], positions[gone], rec[r_halo, :3]]).contiguous()
        q = torch.cat([charges[stay], rec[r_own, 3], charges[gone], rec[r_halo, 3]]).contiguous()
        gid = torch.cat([global_ids[stay], rec[r_own, 4].to(torch.int64), global_ids[gone],
                         rec[r_halo, 4].to(torch.int64)])
        return pos, q, gid, int(n_stay) + int(r_own.sum())

    def _step(self, positions, charges, global_ids, lambdas, n_lambda, sites, n_global, mode):
        torch = self.torch
        if sites is not None and (lambdas is None or n_lambda is None):
            raise ValueError("sites need lambdas and n_lambda (the HI step scales the site charges)")
        d = self.cfg.depth
        pos_l, q_l, gid_l, n_own = self._exchange_particles(positions.contiguous(), charges.contiguous(),
                                                            global_ids)
        n_loc = pos_l.shape[0]
        if self.plan is None:  # positions reach the host once, for the plan's setup
            self._ensure_plan(pos_l.cpu().numpy())
        plan = self.plan
        plan.set_count(n_loc)
        n_sites = 0
        if sites is not None:
            ao, ai, nf, fo, fq = sites
            if self._site_dev is None or self._site_key is not sites:
                self._site_dev = torch.as_tensor(np.asarray(ai, np.int64), device=positions.device)
                self._site_key = sites
                self._site_local = None
            if n_global is None:
                raise ValueError("n_global (the total atom count) is needed with sites")
            loc = torch.full((int(n_global),), -1, dtype=torch.int64, device=positions.device)
            loc[gid_l] = torch.arange(n_loc, device=positions.device)
            ai_l = loc[self._site_dev]
            # re-upload the local site tables only when the local indices moved
            if self._site_local is None or not torch.equal(ai_l, self._site_local):
                plan.set_sites(ao, ai_l.cpu().numpy(), nf, fo, fq)
                self._site_local = ai_l
            n_sites = len(nf)
        plan.dist_phase(1, pos_l, q_l, lambdas if n_sites else None, n_lambda if n_sites else None, grad=True)
        ptrs, loff = plan.dist_buffers()
        # ---- exchange 1: owned multipoles of levels >= lg, dipole / charge ----
        ncp = plan.ncp  # the plan's padded coefficient count (lfmm_dist_buffers)
        tdt = "<f4" if self.tsize == 4 else "<f8"
        for lvl in range(self.lg, d + 1) if self.world > 1 else ():
            nbox = 1 << (3 * lvl)
            view = _device_view(ptrs[0] + int(loff[lvl]) * ncp * self.tsize, (nbox * ncp,), tdt, torch)
            n_l, sh = 1 << lvl, d - lvl
            x0, x1 = self.x0 >> sh, self.x1 >> sh
            if lvl > self.lg and n_l - (x1 - x0) > 2 * HALO_PLANES:
                # M2L sources of the owned targets (children of the parents'
                # neighbours) lie within 2 planes of the slab: halo only
                self.comm.halo_(view, ncp << (2 * lvl), x0, x1, n_l, HALO_PLANES)
            else:
                # level lg (feeds the shared levels' M2M) or a halo that
                # covers every other rank's slab
                self.comm.allgather_(view, nbox * ncp // self.world)
        if ptrs[8] and self.world > 1:
            # fp16 M2L level scales: max over every rank's slab (exact)
            lmax = _device_view(ptrs[8], (d + 1,), "<i4", torch)
            self.comm.max_(lmax)
        if _POISON:
            self._poison(ptrs, loff, ncp, tdt)
        scal = _device_view(ptrs[1], (4,), "<f8", torch)
        scal.copy_(self.comm.sum_ordered(scal.clone()))
        plan.dist_phase(2, grad=True)
        ptrs, _ = plan.dist_buffers()  # phase 2 may (re)allocate the site-potential buffer
        # ---- exchange 2: energies, site potentials, forces ----
        en = _device_view(ptrs[2], (4,), "<f8", torch).clone()
        if _DEBUG:
            torch.cuda.synchronize()
            print("rank", self.rank, "energies", en.cpu().numpy(), "scal", _device_view(ptrs[1], (4,), "<f8", torch).cpu().numpy(), flush=True)
        parts = self.comm.sum_ordered(en[1:3].clone())
        e_solve = float(parts[0] + parts[1] + en[3])
        out = {"energy_solve": e_solve, "near_energy": float(parts[0]), "far_energy": float(parts[1]),
               "dipole_energy": float(en[3]), "owned": gid_l[:n_own], "owned_positions": pos_l[:n_own],
               "owned_charges": q_l[:n_own]}
        if n_sites:
            # site-atom potentials and positions from their owners (each site
            # atom is owned by one rank; the others contribute exact zeros)
            a_tot = int(np.asarray(sites[0])[-1])
            sp = _device_view(ptrs[4], (a_tot,), "<f8", torch)
            ai_l = self._site_local
            mine = (ai_l >= 0) & (ai_l < n_own)
            sp4 = torch.zeros((a_tot, 4), dtype=torch.float64, device=sp.device)
            sp4[:, 3] = sp
            sp4[mine, :3] = pos_l[ai_l[mine]]
            sp4 = self.comm.sum_ordered(sp4)
            sp.copy_(sp4[:, 3])
            plan.dist_hi(sp4[:, :3].contiguous(), mode)
            ptrs, _ = plan.dist_buffers()
            out["lambda_forces"] = _device_view(ptrs[5], (n_sites, 4), "<f8", torch).clone()
            off = float(_device_view(ptrs[6], (1,), "<f8", torch)[0])
            out["energy"] = e_solve + (off if mode == _native.MODE_HI else 0.0)
        else:
            out["energy"] = e_solve
        # after dist_hi: in HI mode the site atoms' rows carry -grad Delta E_site
        out["forces"] = _device_view(ptrs[3], (n_loc, 3), "<f8", torch)[:n_own].clone()
        return out

    def _poison(self, ptrs, loff, ncp, tdt):
        """Test hook (LFMM_DIST_POISON=1): NaN into every multipole plane the
        exchange did not fill, so a read outside the halo shows up in the
        results."""
        torch = self.torch
        d = self.cfg.depth
        for lvl in range(self.lg + 1, d + 1):
            n_l, sh = 1 << lvl, d - lvl
            x0, x1 = self.x0 >> sh, self.x1 >> sh
            if n_l - (x1 - x0) <= 2 * HALO_PLANES:
                continue
            keep = set(range(x0, x1)) | set(halo_planes(x0, x1, n_l, HALO_PLANES))
            view = _device_view(ptrs[0] + int(loff[lvl]) * ncp * self.tsize, (n_l, (ncp << (2 * lvl))), tdt, torch)
            for x in range(n_l):
                if x not in keep:
                    view[x].fill_(float("nan"))

