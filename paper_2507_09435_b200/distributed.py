"""Slab-decomposed implicit MPM Newton step across GPUs.

The reference is single-process: `MpmSim<D>` owns every particle and the whole
grid (/root/reference/proj/include/impm/mpm_solver.hpp:56-477). Its DofMap
numbers nodes in ascending flat order with axis 0 slowest (grid.hpp:30-34,
69-86) and its Jacobian couples nodes within +-2 per axis (jacobian.hpp:36-65),
so an axis-0 slab of node planes is a contiguous range of global DOFs and
Jacobian rows that needs only its own particles, two ghost particle layers and
a 2-plane vector halo. One `SlabSim` per GPU (one process per GPU under
torchrun, NCCL over NVLink / NVSwitch) runs the same Newton controller as the
single-GPU `MpmSim`; all ranks take identical decisions because every norm and
dot product is summed over ranks before use (see csrc/impm_comm.cuh).

Per Newton iteration:  2-plane halo before each SpMV / residual / tangent,
                       elementwise sums of the dot-product partials,
per load step:         allgather of owned DOF counts (global numbering),
                       max particle mass, particle migration to neighbours.

The multigrid preconditioner is rank-local (block Jacobi across slabs), so the
Krylov count may differ slightly from one GPU; the Newton iterates agree to
the Krylov tolerance, and residual / Jacobian rows are bitwise those of the
single-GPU run (same particle order per bin, same colour-batch order).
"""
import ctypes
import threading

import numpy as np

from . import _abi, slabs
from .errors import raise_for
from .particles import GridSpec, ParticleArray, particle_doubles, seed_box_rows
from .sim import DofMap, MaterialSpec, MpmSim, SolverOptions, _Handle

NCCL_ID_BYTES = 128
MIN_PLANES = 4


class Communicator:
    """impm_comm*: NCCL (one process per GPU) or an in-process thread group."""

    def __init__(self, handle):
        L = _abi.lib()
        self._L = L
        self.h = handle
        r, n, k = ctypes.c_int32(), ctypes.c_int32(), ctypes.c_char_p()
        L.impm_comm_info(self.h, ctypes.byref(r), ctypes.byref(n), ctypes.byref(k))
        self.rank, self.nranks, self.kind = r.value, n.value, k.value.decode()

    @classmethod
    def nccl(cls, rank, nranks, device=0, broadcast=None):
        """NCCL communicator; `broadcast(payload_or_None) -> bytes` ships rank 0's
        unique id to the other ranks (e.g. over torch.distributed)."""
        L = _abi.lib()
        idb = None
        if rank == 0:
            buf = (ctypes.c_uint8 * NCCL_ID_BYTES)()
            st = L.impm_comm_nccl_id(buf, NCCL_ID_BYTES)
            if st != _abi.OK:
                raise_for(st, L.impm_create_error().decode())
            idb = bytes(buf)
        if nranks > 1:
            if broadcast is None:
                raise ValueError("nranks > 1 needs a broadcast function for the NCCL unique id")
            idb = broadcast(idb)
        buf = (ctypes.c_uint8 * NCCL_ID_BYTES).from_buffer_copy(idb)
        h = ctypes.c_void_p()
        st = L.impm_comm_nccl_create(buf, rank, nranks, device, ctypes.byref(h))
        if st != _abi.OK:
            raise_for(st, L.impm_create_error().decode())
        return cls(h)

    @classmethod
    def local_group(cls, nranks, device=0):
        """`nranks` communicators for ranks driven by threads of this process on
        one device (host-ordered collectives; the single-GPU test transport)."""
        L = _abi.lib()
        arr = (ctypes.c_void_p * nranks)()
        st = L.impm_comm_local_group(nranks, device, arr)
        if st != _abi.OK:
            raise_for(st, L.impm_create_error().decode())
        return [cls(ctypes.c_void_p(arr[i])) for i in range(nranks)]

    def __del__(self):
        try:
            if getattr(self, "h", None):
                self._L.impm_comm_destroy(self.h)
                self.h = None
        except Exception:
            pass


# ------------------------------------------------------------ geometry --
def slab_cuts(grid: GridSpec, nranks: int, particles=None, use_X=False):
    """Ownership cuts [nranks + 1] along axis 0, balanced by the particle count
    of each bin plane (first support node) when particles are given."""
    n0 = int(grid.nodes[0])
    w = None
    if particles is not None:
        first = slabs.support_first(grid, particles, 0, use_X)
        w = np.bincount(np.clip(first, 0, n0 - 1), minlength=n0)
    return slab_cuts_from_weights(n0, nranks, w)


def slab_cuts_from_weights(n0, nranks, w=None):
    """Cuts balanced by per-plane weights `w` [n0] (None: by plane count)."""
    ranges = slabs.partition_nodes(n0, nranks, w)
    cuts = [r[0] for r in ranges] + [n0]
    if nranks > 1:  # every slab >= MIN_PLANES owned planes (2-plane halos, one-neighbour migration)
        if n0 < MIN_PLANES * nranks:
            from .errors import ConfigError
            raise ConfigError(f"{n0} node planes cannot make {nranks} slabs of >= {MIN_PLANES}")
        for r in range(1, nranks):
            cuts[r] = max(cuts[r], cuts[r - 1] + MIN_PLANES)
        for r in range(nranks - 1, 0, -1):
            cuts[r] = min(cuts[r], cuts[r + 1] - MIN_PLANES)
    return cuts


def slab_extent(n0, cuts, rank):
    """(A, B, lo, hi): owned planes [A, B), local grid planes [lo, hi)."""
    A, B = int(cuts[rank]), int(cuts[rank + 1])
    return A, B, max(0, A - 2), min(int(n0), B + 2)


def keep_mask(first, cuts, rank):
    """Particles rank `rank` holds: first support node in [A - 2, B) (the
    global grid edges keep everything on their open side, so out-of-domain
    particles still reach the reference's OutOfDomainError)."""
    nr = len(cuts) - 1
    A, B = cuts[rank], cuts[rank + 1]
    m = np.ones(first.shape, dtype=bool)
    if rank > 0:
        m &= first >= A - 2
    if rank < nr - 1:
        m &= first < B
    return m


def owned_mask(first, cuts, rank):
    nr = len(cuts) - 1
    A, B = cuts[rank], cuts[rank + 1]
    m = np.ones(first.shape, dtype=bool)
    if rank > 0:
        m &= first >= A
    if rank < nr - 1:
        m &= first < B
    return m


def slab_member_ids(grid: GridSpec, particles, cuts, rank, use_X=False):
    """Global ids (ascending) of the owned + ghost particles of `rank`."""
    first = slabs.support_first(grid, particles, 0, use_X)
    return np.nonzero(keep_mask(first, cuts, rank))[0]


class SlabSim(MpmSim):
    """One slab of a decomposed `MpmSim` (the multi-GPU create variant of the
    C ABI, include/impm_gpu.h `impm_sim_set_slab`). Every call is collective:
    all ranks make the same sequence of calls."""

    def __init__(self, grid: GridSpec, comm: Communicator, cuts, particles, ids, material: MaterialSpec,
                 options=None, device: int = 0):
        self.global_grid = grid
        self.comm = comm
        self.cuts = [int(c) for c in cuts]
        if len(self.cuts) != comm.nranks + 1:
            raise ValueError("cuts must have nranks + 1 entries")
        n0 = int(grid.nodes[0])
        self.A, self.B, self.lo, self.hi = slab_extent(n0, self.cuts, comm.rank)
        local = GridSpec(grid.dim, tuple(grid.origin), grid.h, (self.hi - self.lo,) + tuple(grid.nodes[1:grid.dim]))
        # MpmSim state, built by hand: the C grid keeps the GLOBAL origin (the
        # slab's node i sits at origin + (lo + i) h, bitwise as on one GPU)
        self.grid = local
        self.D = grid.dim
        self.material = material
        self.options = options or SolverOptions()
        self._h = _Handle(local, material, self.options, device)
        self._N = local.node_count()
        self.fixed = np.zeros(self._N * self.D, dtype=np.uint8)
        self._fixed_sent = None
        self._gravity = np.zeros(self.D)
        cuts_arr = np.asarray(self.cuts, dtype=np.int32)
        self._h.call("impm_sim_set_slab", comm.h, n0, _abi.ptr(cuts_arr))
        self.set_particles(particles, ids)
        self._push_gravity()

    @classmethod
    def from_global(cls, grid, comm, cuts, particles, material, options=None, device=0):
        """Slab of a global particle array (ids = row index in it)."""
        data = particles.data if isinstance(particles, ParticleArray) else np.asarray(particles, dtype=np.float64)
        use_X = bool(options and options.total_lagrangian)
        ids = slab_member_ids(grid, data, cuts, comm.rank, use_X)
        return cls(grid, comm, cuts, np.ascontiguousarray(data[ids]), ids, material, options, device)

    # ------------------------------------------------------------ particles
    def set_particles(self, particles, ids=None):
        data = particles.data if isinstance(particles, ParticleArray) else np.asarray(particles, dtype=np.float64)
        data = np.ascontiguousarray(data, dtype=np.float64)
        if data.ndim != 2 or data.shape[1] != particle_doubles(self.D):
            raise ValueError(f"particles must be (P, {particle_doubles(self.D)}) float64")
        if ids is None:
            raise ValueError("slab particles need their global ids")
        ids = np.ascontiguousarray(ids, dtype=np.int64)
        self._h.call("impm_sim_set_particles_ids", _abi.ptr(data), _abi.ptr(ids), data.shape[0], 8 * data.shape[1])

    @property
    def n_particles(self):
        n = ctypes.c_int64()
        self._h.call("impm_sim_n_particles", ctypes.byref(n))
        return n.value

    @property
    def particles(self):
        raise AttributeError("a slab holds owned + ghost particles: use local_particles() / owned_particles()")

    def local_particles(self):
        """(ParticleArray, ids) of every particle this rank holds, local order."""
        P = self.n_particles
        out = np.zeros((P, particle_doubles(self.D)), dtype=np.float64)
        ids = np.zeros(max(P, 1), dtype=np.int64)
        self._h.call("impm_sim_get_particles_ids", _abi.ptr(out), _abi.ptr(ids), P, 8 * out.shape[1])
        return ParticleArray(out, self.D), ids[:P]

    def owned_particles(self):
        """(ParticleArray, ids) of the particles this rank owns (first support
        node in [A, B) at the current configuration)."""
        pa, ids = self.local_particles()
        first = slabs.support_first(self.global_grid, pa.data, 0, bool(self.options.total_lagrangian))
        m = owned_mask(first, self.cuts, self.comm.rank)
        return ParticleArray(np.ascontiguousarray(pa.data[m]), self.D), ids[m]

    # ------------------------------------------------------------ grid
    def node_positions(self):
        """Global coordinates of the local nodes (origin + global index * h)."""
        g = self.grid
        idx = np.indices([int(n) for n in g.nodes[: g.dim]]).reshape(g.dim, -1).T
        idx[:, 0] += self.lo
        return np.asarray(g.origin[: g.dim], dtype=np.float64) + idx * g.h

    def global_node_ids(self):
        """Global flat index of every local node (local flat order)."""
        inner = int(np.prod(self.global_grid.nodes[1:self.D])) if self.D > 1 else 1
        return ((np.arange(self.hi - self.lo)[:, None] + self.lo) * inner + np.arange(inner)[None, :]).reshape(-1)

    def owned_node_mask(self):
        inner = int(np.prod(self.global_grid.nodes[1:self.D])) if self.D > 1 else 1
        i0 = np.repeat(np.arange(self.lo, self.hi), inner)
        return (i0 >= self.A) & (i0 < self.B)

    def fix_nodes(self, predicate, component=-1):
        pos = self.node_positions()
        mask = np.asarray(predicate(pos), dtype=bool).reshape(-1)
        for c in range(self.D):
            if component < 0 or component == c:
                self.fixed[np.nonzero(mask)[0] * self.D + c] = 1

    def set_fixed_global(self, fixed_global):
        """Slice of the global `fixed` array ([node*D + comp])."""
        fg = np.asarray(fixed_global, dtype=np.uint8).reshape(-1, self.D)
        self.fixed = np.ascontiguousarray(fg[self.global_node_ids()].reshape(-1))

    # ------------------------------------------------------------ DOFs
    def slab_info(self):
        n, off, b = ctypes.c_int64(), ctypes.c_int64(), ctypes.c_int32()
        self._h.call("impm_sim_slab_info", ctypes.byref(n), ctypes.byref(off), ctypes.byref(b))
        return {"n_dofs_global": n.value, "dof_offset": off.value, "base0": b.value}

    def global_dofs(self):
        """(global node ids of the owned nodes, their global dof_of [.., D]):
        the local DofMap of the owned nodes shifted by this rank's offset."""
        dm: DofMap = self.dofs()
        off = self.slab_info()["dof_offset"]
        own = self.owned_node_mask()
        d = dm.dof_of.reshape(-1, self.D)[own]
        return self.global_node_ids()[own], np.where(d >= 0, d + off, -1)

    # ------------------------------------------------------------ stepping
    def migrate(self):
        self._h.call("impm_sim_migrate")

    # step(): impm_sim_step = begin_step + newton_solve + commit_step + migrate


def run_local_ranks(nranks, fn, device=0, timeout=900):
    """Runs fn(rank, comm) for every rank of an in-process group, one host
    thread per rank on one device (ctypes releases the GIL inside the C ABI);
    returns the per-rank results, re-raising the first failure."""
    comms = Communicator.local_group(nranks, device)
    out, errs = [None] * nranks, [None] * nranks

    def body(r):
        try:
            out[r] = fn(r, comms[r])
        except BaseException as e:  # noqa: BLE001 - reported below
            errs[r] = e

    ts = [threading.Thread(target=body, args=(r,), daemon=True) for r in range(nranks)]
    for t in ts:
        t.start()
    for t in ts:
        t.join(timeout)
    if any(t.is_alive() for t in ts):
        raise TimeoutError("a slab rank did not finish (collective mismatch?)")
    for e in errs:
        if e is not None:
            raise e
    return out


def gather_owned(results, D):
    """Concatenates per-rank (ParticleArray, ids) of owned particles in
    global-id order."""
    datas = [r[0].data for r in results]
    ids = np.concatenate([r[1] for r in results])
    order = np.argsort(ids, kind="stable")
    return ParticleArray(np.concatenate(datas)[order], D), ids[order]


def seed_box_slab(grid: GridSpec, lo, hi, ppc, density, cuts, rank, use_X=False):
    """The rows of seed_box(grid, lo, hi, ppc, density) that rank `rank` holds,
    generated without the global array: (particles, global ids)."""
    D = grid.dim
    cells = [int(np.floor((hi[a] - lo[a]) / grid.h + 0.5)) for a in range(D)]
    sub0 = cells[0] * ppc
    spacing = grid.h / ppc
    x0 = lo[0] + (np.arange(sub0, dtype=np.float64) + 0.5) * spacing
    lp = np.full(sub0, 0.5 * spacing)
    first = np.floor((x0 - grid.origin[0] - (grid.h + lp)) / grid.h).astype(np.int64) + 1
    rows = np.nonzero(keep_mask(first, cuts, rank))[0]
    return seed_box_rows(grid, lo, hi, ppc, density, rows)
