"""Device-resident scene state S = {G, C} (reference `pkg/src/contrags/model.py`).

Per-Gaussian arrays and codebook rows live in HBM as torch tensors carved
from capacity-headroom buffers (so densify and row appends do not
reallocate every step); the MCMC bookkeeping the host decides on --
refcounts, split-lineage parents and the min-heap free list -- lives in
host numpy mirrors with the reference's exact semantics
(`model.py:33-118`).  A device int32 copy of the refcounts is uploaded
lazily for the kernels that need it.
"""

from __future__ import annotations

import heapq

import numpy as np
import torch

SR_DIM = 7  # model.py:16


def sh_dim(degree: int) -> int:
    """model.py:19-23"""
    if degree not in (0, 1, 2, 3):
        raise ValueError(f"sh_degree must be in 0..3, got {degree}")
    return 3 * (degree + 1) ** 2


def degree_from_dim(dim: int) -> int:
    """model.py:26-30"""
    for deg in (0, 1, 2, 3):
        if sh_dim(deg) == dim:
            return deg
    raise ValueError(f"SH codebook dim {dim} does not match any degree 0..3")


def default_device():
    if not torch.cuda.is_available():
        raise RuntimeError("paper_2509_03775_b200 needs a CUDA device (B200, sm_100a); "
                           "there is no CPU fallback")
    return torch.device("cuda", torch.cuda.current_device())


def _grow(buf: torch.Tensor, need: int) -> torch.Tensor:
    if buf.shape[0] >= need:
        return buf
    new_cap = max(need, int(buf.shape[0] * 1.5) + 16)
    nb = torch.empty((new_cap,) + tuple(buf.shape[1:]), dtype=buf.dtype, device=buf.device)
    nb[: buf.shape[0]] = buf
    return nb


class Codebook:
    """Shared-row store: device rows, host refcount / parent / free heap.

    Same contract as reference `Codebook` (model.py:33-118): rows (capacity,
    dim) float32; dead rows stay in place; alloc reuses the lowest free index,
    else appends one row; decref to zero frees the row, clears its parent and
    breaks lineage into it.
    """

    def __init__(self, rows, device=None, headroom: float = 0.25):
        dev = torch.device(device) if device is not None else default_device()
        if isinstance(rows, torch.Tensor):
            r = rows.detach().to(device=dev, dtype=torch.float32)
        else:
            r = torch.as_tensor(np.ascontiguousarray(rows, dtype=np.float32), device=dev)
        if r.dim() != 2:
            raise ValueError("codebook rows must be 2-D")
        cap = r.shape[0]
        self._buf = torch.empty((cap + int(cap * headroom) + 16, r.shape[1]), dtype=torch.float32,
                                device=dev)
        self._buf[:cap] = r
        self._cap = cap
        self._rc = np.zeros(cap, dtype=np.int64)
        self._pending = []  # deferred refcount updates (device densify), see refcount
        self.parent = np.full(cap, -1, dtype=np.int32)
        self._free: list = []
        self._dev_rc = None
        self._dev_rc_host = None
        self._live_cache = None
        self._live_version = 0  # bumped whenever the free heap (the dead rows) changes
        self.mutations = 0

    # -- host refcount mirror ----------------------------------------------
    @property
    def refcount(self) -> np.ndarray:
        """Host refcounts (model.py:41-48).  A device-side densify leaves its
        increments pending until the next host read (applied here, in order),
        so training steps never wait for the device."""
        if self._pending:
            fns, self._pending = self._pending, []
            for fn in fns:
                fn(self._rc)
        return self._rc

    @refcount.setter
    def refcount(self, value):
        self._pending = []
        self._rc = value

    # -- shape ------------------------------------------------------------
    @property
    def rows(self) -> torch.Tensor:
        return self._buf[: self._cap]

    @rows.setter
    def rows(self, value):
        t = value if isinstance(value, torch.Tensor) else torch.as_tensor(np.asarray(value, np.float32))
        t = t.to(device=self._buf.device, dtype=torch.float32)
        if t.shape[0] > self._buf.shape[0] or t.shape[1] != self._buf.shape[1]:
            self._buf = torch.empty((t.shape[0] + 16, t.shape[1]), dtype=torch.float32,
                                    device=self._buf.device)
        self._buf[: t.shape[0]] = t
        self._cap = t.shape[0]
        self.mutations += 1

    @property
    def device(self):
        return self._buf.device

    @property
    def dim(self) -> int:
        return int(self._buf.shape[1])

    @property
    def capacity(self) -> int:
        return self._cap

    @property
    def live_count(self) -> int:
        return self.capacity - len(self._free)

    @property
    def free_set(self) -> set:
        return set(self._free)

    def is_live(self, r: int) -> bool:
        return 0 <= r < self.capacity and self.refcount[r] > 0

    def live_indices(self) -> np.ndarray:
        return np.flatnonzero(self.refcount > 0)

    def row(self, r: int) -> np.ndarray:
        if not self.is_live(r):
            raise ValueError(f"codebook row {r} is not live")
        return self.rows[r].detach().cpu().numpy().copy()

    # -- bookkeeping (model.py:78-118) -----------------------------------
    def alloc(self, value, parent: int = -1) -> int:
        v = np.asarray(value.detach().cpu().numpy() if isinstance(value, torch.Tensor) else value,
                       dtype=np.float32)
        if v.shape != (self.dim,):
            raise ValueError(f"row value must have shape ({self.dim},)")
        r = self.alloc_index(parent)
        self._buf[r] = torch.as_tensor(v, device=self._buf.device)
        return r

    def alloc_index(self, parent: int = -1) -> int:
        """Allocate a row index (refcount 1) without writing its value."""
        if parent != -1 and not self.is_live(parent):
            raise ValueError(f"parent row {parent} is not live")
        self._live_version += 1
        if self._free:
            r = heapq.heappop(self._free)
        else:
            r = self._cap
            self._buf = _grow(self._buf, r + 1)
            self._cap = r + 1
            self.refcount = np.concatenate([self.refcount, [0]])
            self.parent = np.concatenate([self.parent, [-1]]).astype(np.int32)
        self.refcount[r] = 1
        self.parent[r] = parent
        self.mutations += 1
        return r

    def incref(self, r: int) -> None:
        if not self.is_live(r):
            raise ValueError(f"cannot reference dead row {r}")
        self.refcount[r] += 1
        self.mutations += 1

    def decref(self, r: int) -> bool:
        if not self.is_live(r):
            raise ValueError(f"cannot release dead row {r}")
        self.refcount[r] -= 1
        self.mutations += 1
        if self.refcount[r] == 0:
            self.parent[r] = -1
            self.parent[self.parent == r] = -1
            heapq.heappush(self._free, int(r))
            self._live_version += 1
            return True
        return False

    def lineage_pairs(self) -> np.ndarray:
        children = np.flatnonzero((self.parent >= 0) & (self.refcount > 0))
        if len(children) == 0:
            return np.zeros((0, 2), dtype=np.int64)
        return np.stack([children, self.parent[children]], axis=1)

    def reset_free_list(self):
        """Rebuild the free heap from zero refcounts (after bulk refcount edits)."""
        self._free = [int(r) for r in np.flatnonzero(self.refcount == 0)]
        heapq.heapify(self._free)
        self._live_version += 1

    # -- device mirrors ---------------------------------------------------
    def device_refcount(self) -> torch.Tensor:
        """int32 device copy of the host refcounts (uploaded when they changed)."""
        if (self._dev_rc is None or self._dev_rc_host is None
                or self._dev_rc_host.shape != self.refcount.shape
                or not np.array_equal(self._dev_rc_host, self.refcount)):
            from . import _native as nat
            self._dev_rc = nat.upload(self.refcount, self._buf.device, np.int32)
            self._dev_rc_host = self.refcount.copy()
        return self._dev_rc

    def device_live(self) -> torch.Tensor:
        """int32 device list of live row indices, ascending.  Reads the refcounts
        without applying pending densify increments: those only raise counts of
        rows that are already live, so the live set is the same (and the
        training loop does not wait for the device)."""
        # the live rows are exactly the rows not in the free heap (validate_state):
        # its size, identity and change counter key the cache (O(1), no scan)
        key = (self._cap, len(self._free), id(self._free), self._live_version)
        if self._live_cache is None or self._live_cache[0] != key:
            from . import _native as nat
            self._live_cache = (key, nat.upload(np.flatnonzero(self._rc > 0), self._buf.device,
                                                np.int32))
        return self._live_cache[1]


class GaussianArrays:
    """Per-Gaussian device arrays sharing length N (reference model.py:121-135).

    Backed by capacity buffers; the public attributes are length-N views.
    Assigning an attribute (numpy or torch) replaces its contents.
    """

    _FIELDS = ("positions", "opacity_logits", "g2sh", "g2sr")

    def __init__(self, positions, opacity_logits, g2sh, g2sr, device=None, headroom: float = 0.0):
        dev = torch.device(device) if device is not None else default_device()
        self._dev = dev
        n = len(positions)
        cap = n + int(n * headroom)
        self._pos = torch.empty((cap, 3), dtype=torch.float32, device=dev)
        self._logit = torch.empty((cap,), dtype=torch.float32, device=dev)
        self._g2sh = torch.empty((cap,), dtype=torch.int32, device=dev)
        self._g2sr = torch.empty((cap,), dtype=torch.int32, device=dev)
        self._n = n
        self.positions = positions
        self.opacity_logits = opacity_logits
        self.g2sh = g2sh
        self.g2sr = g2sr

    def _to(self, v, dtype):
        if isinstance(v, torch.Tensor):
            return v.detach().to(device=self._dev, dtype=dtype)
        npd = np.float32 if dtype == torch.float32 else np.int32
        return torch.as_tensor(np.ascontiguousarray(v, dtype=npd)).to(self._dev)

    def _set(self, name, value, dtype, width):
        t = self._to(value, dtype)
        n = t.shape[0]
        if n != self._n:
            self.resize(n)
        buf = getattr(self, name)
        buf[:n] = t.reshape((n, width)) if width > 1 else t.reshape(n)

    def resize(self, n: int):
        """Change N (keeps the first min(N, n) entries), growing buffers if needed."""
        for name in ("_pos", "_logit", "_g2sh", "_g2sr"):
            setattr(self, name, _grow(getattr(self, name), n))
        self._n = n

    def reserve(self, cap: int):
        for name in ("_pos", "_logit", "_g2sh", "_g2sr"):
            setattr(self, name, _grow(getattr(self, name), cap))

    @property
    def positions(self):
        return self._pos[: self._n]

    @positions.setter
    def positions(self, v):
        self._set("_pos", v, torch.float32, 3)

    @property
    def opacity_logits(self):
        return self._logit[: self._n]

    @opacity_logits.setter
    def opacity_logits(self, v):
        self._set("_logit", v, torch.float32, 1)

    @property
    def g2sh(self):
        return self._g2sh[: self._n]

    @g2sh.setter
    def g2sh(self, v):
        self._set("_g2sh", v, torch.int32, 1)

    @property
    def g2sr(self):
        return self._g2sr[: self._n]

    @g2sr.setter
    def g2sr(self, v):
        self._set("_g2sr", v, torch.int32, 1)

    @property
    def count(self) -> int:
        return self._n

    @property
    def capacity(self) -> int:
        """Rows allocated in the backing buffers (N can grow to this in place)."""
        return int(self._pos.shape[0])

    def opacities(self) -> np.ndarray:
        """sigmoid(logit) in float64 on the host (model.py:134-135)."""
        lg = self.opacity_logits.detach().cpu().numpy().astype(np.float64)
        return 1.0 / (1.0 + np.exp(-lg))


class ModelState:
    """Full compressed scene (reference model.py:138-154), device-resident."""

    def __init__(self, gaussians: GaussianArrays, sh: Codebook, sr: Codebook, iteration: int = 0,
                 rng_seed: int = 0):
        self.gaussians = gaussians
        self.sh = sh
        self.sr = sr
        self.iteration = iteration
        self.rng_seed = rng_seed
        self.mutations = 0
        self.assign_version = 0

    @property
    def num_gaussians(self) -> int:
        return self.gaussians.count

    @property
    def sh_degree(self) -> int:
        return degree_from_dim(self.sh.dim)

    @property
    def device(self):
        return self.sh.device

    def touch(self, assignments: bool = False):
        """Record an in-place mutation made by a kernel (staleness token).

        ``assignments`` marks a change of g2sh / g2sr (invalidates the code CSRs).
        """
        self.mutations += 1
        if assignments:
            self.assign_version += 1

    def code_csr(self, which: str):
        """(offsets (cap+1,), members (N,)) int32 device CSR of one index array.

        Cached; rebuilt (cgs_code_csr: one stable onesweep) only when the
        assignments, N or the capacity changed.
        """
        from . import _native as nat
        book, idx = _book_of(self, which)
        key = (self.assign_version, idx.data_ptr(), idx._version, idx.shape[0], book.capacity)
        cache = self.__dict__.setdefault("_csr", {})
        hit = cache.get(which)
        if hit is not None and hit[0] == key:
            return hit[1], hit[2]
        n, cap = idx.shape[0], book.capacity
        off = torch.empty((cap + 1,), dtype=torch.int32, device=book.device)
        mem = torch.empty((max(n, 1),), dtype=torch.int32, device=book.device)
        nb = nat.library().cgs_code_csr_workspace_bytes(max(n, 1), cap)
        ws = torch.empty((nb,), dtype=torch.uint8, device=book.device)
        nat.call("cgs_code_csr", nat.ptr(idx), n, cap, nat.ptr(off), nat.ptr(mem), nat.ptr(ws),
                 nb, nat.stream_handle(book.device))
        cache[which] = (key, off, mem)
        return off, mem

    # -- host mirror of the assignments -------------------------------------
    # g2sh / g2sr change only through host-decided moves (split, merge,
    # densify, remap), so the MCMC decision loop reads them from a host copy
    # fetched asynchronously right after each change instead of synchronising
    # with the device at the next transition.
    def _index_key(self, which):
        _, idx = _book_of(self, which)
        return (self.assign_version, idx.data_ptr(), idx._version, idx.shape[0])

    def prefetch_host_index(self, which=None):
        """Enqueue a pinned D2H copy of g2sh / g2sr on the current stream."""
        cache = self.__dict__.setdefault("_hidx", {})
        for w in (("sh", "sr") if which is None else (which,)):
            key = self._index_key(w)
            ent = cache.get(w)
            if ent is not None and ent[0] == key:
                continue
            _, idx = _book_of(self, w)
            # one pinned buffer per index array, sized for the Gaussian capacity
            # and reused (a new pinned allocation per densify costs milliseconds)
            pool = self.__dict__.setdefault("_hidx_buf", {})
            buf = pool.get(w)
            if buf is None or buf.numel() < idx.shape[0]:
                cap = max(idx.shape[0], self.gaussians.capacity)
                buf = torch.empty((cap,), dtype=torch.int32, pin_memory=idx.is_cuda)
                pool[w] = buf
            host = buf[: idx.shape[0]]  # copies into buf are ordered on the stream
            host.copy_(idx, non_blocking=True)
            ev = None
            if idx.is_cuda:
                ev = torch.cuda.Event()
                ev.record()
            cache[w] = (key, host, ev)

    def host_index(self, which: str) -> np.ndarray:
        """int32 host copy of g2sh ('sh') or g2sr ('sr'), current with the device."""
        self.prefetch_host_index(which)
        key, host, ev = self.__dict__["_hidx"][which]
        if ev is not None:
            ev.synchronize()
        return host.numpy()

    def token(self) -> tuple:
        """Cheap identity of the state contents (replaces render.py:227-237's SHA-256)."""
        g = self.gaussians
        ts = (g.positions, g.opacity_logits, g.g2sh, g.g2sr, self.sh.rows, self.sr.rows)
        # rendering does not read refcounts; their host-side changes all bump
        # a mutation counter
        return (self.mutations, self.sh.mutations, self.sr.mutations,
                tuple((t.data_ptr(), t.shape[0], t._version) for t in ts))

    # -- construction -----------------------------------------------------
    @classmethod
    def from_arrays(cls, positions, opacity_logits, g2sh, g2sr, sh_rows, sr_rows,
                    sh_refcount=None, sr_refcount=None, sh_parent=None, sr_parent=None,
                    device=None, iteration: int = 0, rng_seed: int = 0,
                    gaussian_headroom: float = 0.0) -> "ModelState":
        """State from host arrays; refcounts default to bincount, free heap = zero rows."""
        g2sh = np.asarray(g2sh, dtype=np.int32)
        g2sr = np.asarray(g2sr, dtype=np.int32)
        sh = Codebook(sh_rows, device=device)
        sr = Codebook(sr_rows, device=device)
        for book, idx, rc, par in ((sh, g2sh, sh_refcount, sh_parent), (sr, g2sr, sr_refcount, sr_parent)):
            book.refcount = (np.bincount(idx, minlength=book.capacity).astype(np.int64)
                             if rc is None else np.asarray(rc, np.int64).copy())
            if par is not None:
                book.parent = np.asarray(par, np.int32).copy()
            book.reset_free_list()
        ga = GaussianArrays(positions, opacity_logits, g2sh, g2sr, device=sh.device,
                            headroom=gaussian_headroom)
        return cls(ga, sh, sr, iteration=iteration, rng_seed=rng_seed)

    def to_host(self) -> dict:
        """Host copies of every array (for checks and serialization)."""
        g = self.gaussians
        return dict(positions=g.positions.cpu().numpy(), opacity_logits=g.opacity_logits.cpu().numpy(),
                    g2sh=g.g2sh.cpu().numpy(), g2sr=g.g2sr.cpu().numpy(),
                    sh_rows=self.sh.rows.cpu().numpy(), sr_rows=self.sr.rows.cpu().numpy(),
                    sh_refcount=self.sh.refcount.copy(), sr_refcount=self.sr.refcount.copy(),
                    sh_parent=self.sh.parent.copy(), sr_parent=self.sr.parent.copy(),
                    sh_free=np.array(sorted(self.sh._free), dtype=np.int64),
                    sr_free=np.array(sorted(self.sr._free), dtype=np.int64))


def init_one_to_one(n: int, sh_degree: int, seed: int,
                    position_box=((-1.0, -1.0, -1.0), (1.0, 1.0, 1.0)), device=None) -> ModelState:
    """One private row per Gaussian (reference model.py:157-198, same draws)."""
    if n < 1:
        raise ValueError(f"n must be >= 1, got {n}")
    dim = sh_dim(sh_degree)
    lo = np.asarray(position_box[0], dtype=np.float64)
    hi = np.asarray(position_box[1], dtype=np.float64)
    if lo.shape != (3,) or hi.shape != (3,) or np.any(hi <= lo):
        raise ValueError("position_box must be ((x0,y0,z0), (x1,y1,z1)) with hi > lo")
    rng = np.random.default_rng(seed)
    positions = rng.uniform(lo, hi, size=(n, 3)).astype(np.float32)
    sh_rows = np.zeros((n, dim), dtype=np.float32)
    sh_rows[:, 0:3] = rng.uniform(-0.5, 0.5, size=(n, 3)).astype(np.float32)
    sr_rows = np.zeros((n, SR_DIM), dtype=np.float32)
    sr_rows[:, 0:3] = np.log(0.01 * float(np.linalg.norm(hi - lo)))
    sr_rows[:, 3] = 1.0
    idx = np.arange(n, dtype=np.int32)
    st = ModelState.from_arrays(positions, np.zeros(n, np.float32), idx, idx, sh_rows, sr_rows,
                                device=device, rng_seed=seed)
    return st


def _book_of(state: ModelState, which: str):
    if which == "sh":
        return state.sh, state.gaussians.g2sh
    if which == "sr":
        return state.sr, state.gaussians.g2sr
    raise ValueError(f"codebook name must be 'sh' or 'sr', got {which!r}")


def lookup(state: ModelState, i: int):
    """(sh_row, sr_row) backing Gaussian i (model.py:201-206)."""
    if not 0 <= i < state.num_gaussians:
        raise ValueError(f"gaussian index {i} out of range for N={state.num_gaussians}")
    return (state.sh.row(int(state.gaussians.g2sh[i])), state.sr.row(int(state.gaussians.g2sr[i])))


def remap_gaussian(state: ModelState, i: int, which: str, new_row: int) -> None:
    """model.py:209-224"""
    if not 0 <= i < state.num_gaussians:
        raise ValueError(f"gaussian index {i} out of range for N={state.num_gaussians}")
    book, idx = _book_of(state, which)
    old = int(idx[i])
    if new_row == old:
        return
    if not book.is_live(new_row):
        raise ValueError(f"target row {new_row} is not live")
    book.incref(new_row)
    idx[i] = int(new_row)
    book.decref(old)
    state.touch(assignments=True)


def _add_counts(rc: np.ndarray, rows: np.ndarray) -> None:
    """rc[r] += (occurrences of r in rows), in place (== np.add.at(rc, rows, 1),
    ~10x faster for the 5% of N clones a densify adds)."""
    rc += np.bincount(rows, minlength=len(rc))[: len(rc)].astype(rc.dtype, copy=False)


def densify(state: ModelState, growth_rate: float, cap: int, rng: np.random.Generator,
            jitter_sigma: float = 0.02, device_select: bool = False) -> int:
    """Opacity-proportional cloning with shared rows (model.py:235-267).

    Parity mode (default): the host draws exactly the reference's `choice`
    and `normal` sequence from the opacities (one device read); the append
    runs on the device (cgs_densify_append).  ``device_select`` (throughput
    mode, the trainer with device noise): the host draws the same uniforms
    and normals without reading the device, the selection runs on the device
    (cgs_densify_select) and the refcount increments are applied from the
    refreshed assignment mirror when the host next reads refcounts -- no
    synchronisation in the training loop.
    """
    from . import _native as nat
    if growth_rate <= 0:
        raise ValueError("growth_rate must be positive")
    g = state.gaussians
    n = g.count
    if cap < n:
        raise ValueError(f"cap {cap} is below current count {n}")
    k = min(int(growth_rate * n), cap - n)
    if k <= 0:
        return 0
    if device_select:
        return _densify_device(state, n, k, rng, jitter_sigma)
    hsh, hsr = state.host_index("sh"), state.host_index("sr")
    opac = g.opacities()
    probs = opac / opac.sum()
    src = rng.choice(n, size=k, replace=True, p=probs)
    jitter = rng.normal(0.0, jitter_sigma, size=(k, 3))
    dev = state.device
    g.resize(n + k)
    src_d = nat.upload(src, dev, np.int64)
    jit_d = nat.upload(jitter, dev, np.float64)
    nat.call("cgs_densify_append", nat.ptr(g._pos), nat.ptr(g._logit), nat.ptr(g._g2sh),
             nat.ptr(g._g2sr), n, nat.ptr(src_d), nat.ptr(jit_d), k, nat.stream_handle(dev))
    new_sh, new_sr = hsh[src], hsr[src]  # clones share their source's rows (model.py:262-266)
    _add_counts(state.sh.refcount, new_sh)
    _add_counts(state.sr.refcount, new_sr)
    state.sh.mutations += 1
    state.sr.mutations += 1
    state.touch(assignments=True)
    state.prefetch_host_index()
    return k


class _DensifyBuffers:
    """Device and pinned host buffers of the throughput-mode densify, kept
    with the state and grown only when a draw needs more (a first-use pinned
    or device allocation inside a training window cost 35-97 ms at N=1M)."""

    def __init__(self):
        self.k = self.n = 0
        self.ev = None

    def ensure(self, n: int, k: int, dev):
        from . import _native as nat
        if k > self.k:
            self.k = max(k, int(self.k * 1.25))
            self.u_h = torch.empty((self.k,), dtype=torch.float64, pin_memory=True)
            self.jit_h = torch.empty((self.k, 3), dtype=torch.float64, pin_memory=True)
            self.u_d = torch.empty((self.k,), dtype=torch.float64, device=dev)
            self.jit_d = torch.empty((self.k, 3), dtype=torch.float64, device=dev)
            self.src_d = torch.empty((self.k,), dtype=torch.int64, device=dev)
        if n > self.n:
            self.n = max(n, int(self.n * 1.25))
            nb = nat.library().cgs_densify_select_workspace_bytes(self.n)
            self.ws = torch.empty((nb,), dtype=torch.uint8, device=dev)
        return self


def densify_prepare(state: ModelState, n: int, k: int) -> None:
    """Allocate the throughput-mode densify buffers for up to ``n`` Gaussians
    and ``k`` clones ahead of time (the trainer does, for its capacity)."""
    if not hasattr(state, "_densify_bufs"):
        state._densify_bufs = _DensifyBuffers()
    state._densify_bufs.ensure(n, k, state.device)


def _densify_device(state: ModelState, n: int, k: int, rng, jitter_sigma: float) -> int:
    from . import _native as nat
    g = state.gaussians
    dev = state.device
    u = rng.random(k)  # == the uniforms numpy's choice(n, k, p=...) draws
    jitter = rng.normal(0.0, jitter_sigma, size=(k, 3))
    g.resize(n + k)
    densify_prepare(state, n, k)
    b = state._densify_bufs
    if b.ev is not None:
        b.ev.synchronize()  # the previous densify's uploads have left the pinned buffers
    b.u_h[:k].numpy()[:] = u
    b.jit_h[:k].numpy()[:] = jitter
    u_d, jit_d, src_d = b.u_d[:k], b.jit_d[:k], b.src_d[:k]
    u_d.copy_(b.u_h[:k], non_blocking=True)
    jit_d.copy_(b.jit_h[:k], non_blocking=True)
    b.ev = torch.cuda.Event()
    b.ev.record()
    nb, ws = b.ws.numel(), b.ws
    st = nat.stream_handle(dev)
    nat.call("cgs_densify_select", nat.ptr(g._logit), n, nat.ptr(u_d), k, nat.ptr(src_d),
             nat.ptr(ws), nb, st)
    nat.call("cgs_densify_append", nat.ptr(g._pos), nat.ptr(g._logit), nat.ptr(g._g2sh),
             nat.ptr(g._g2sr), n, nat.ptr(src_d), nat.ptr(jit_d), k, st)
    state.sh.mutations += 1
    state.sr.mutations += 1
    state.touch(assignments=True)
    state.prefetch_host_index()  # includes the clones' rows [n, n + k)
    for which, book in (("sh", state.sh), ("sr", state.sr)):
        book._pending.append(
            lambda rc, w=which: _add_counts(rc, state.host_index(w)[n:n + k]))
    return k


def model_bytes(state: ModelState):
    """model.py:270-283"""
    n = state.num_gaussians
    if n == 0:
        return 0, 0, 1.0
    dim = state.sh.dim
    compressed = n * (3 * 4 + 4 + 4 + 4) + state.sh.live_count * dim * 4 + state.sr.live_count * SR_DIM * 4
    dense = n * (3 + 1 + dim + SR_DIM) * 4
    return compressed, dense, dense / compressed


def validate_state(state: ModelState) -> None:
    """All structural invariants (model.py:286-316); refcounts via a device histogram."""
    from . import _native as nat
    g = state.gaussians
    n = g.count
    for name, arr in (("opacity_logits", g.opacity_logits), ("g2sh", g.g2sh), ("g2sr", g.g2sr)):
        if arr.shape[0] != n:
            raise ValueError(f"{name} has length {arr.shape[0]}, expected {n}")
    for which, book, idx in (("sh", state.sh, g.g2sh), ("sr", state.sr, g.g2sr)):
        if n:
            lo, hi = int(idx.min()), int(idx.max())
            if lo < 0 or hi >= book.capacity:
                raise ValueError(f"{which} index out of range")
        counts = torch.empty(max(book.capacity, 1), dtype=torch.int32, device=book.device)
        nat.call("cgs_refcount_histogram", nat.ptr(idx), n, nat.ptr(counts), book.capacity,
                 nat.stream_handle(book.device))
        counted = counts[: book.capacity].cpu().numpy().astype(np.int64)
        if not np.array_equal(counted, book.refcount):
            raise ValueError(f"{which} refcounts disagree with the index arrays")
        if book.free_set != set(np.flatnonzero(book.refcount == 0).tolist()):
            raise ValueError(f"{which} free list disagrees with zero refcounts")
        lp = book.parent[book.refcount > 0]
        lp = lp[lp >= 0]
        if len(lp) and np.any(book.refcount[lp] == 0):
            raise ValueError(f"{which} has a live row whose parent is dead")
        for start in np.flatnonzero((book.parent >= 0) & (book.refcount > 0)):
            seen = set()
            r = int(start)
            while r != -1:
                if r in seen:
                    raise ValueError(f"{which} parent chain starting at {start} cycles")
                seen.add(r)
                r = int(book.parent[r])
    if int(state.sh.refcount.sum()) != n or int(state.sr.refcount.sum()) != n:
        raise ValueError("total refcounts do not equal the Gaussian count")
