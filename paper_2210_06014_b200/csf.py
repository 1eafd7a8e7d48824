"""Balanced compressed-sparse-fiber (B-CSF) trees, built on the GPU (kernel K1).

Mirrors csf.CsfTree / CsfForest / build_tree / build_forest
(/root/reference/pkg/src/fastertucker/csf.py:32-201).  The tree rooted at mode t stores
coordinates in level order (t, t+1, ..., t+N-1) mod N; fibers are runs of equal first N-1
levels; a root slice holding more than ``fiber_threshold`` fibers is split into consecutive
subtensors of at most that many whole fibers.  Every array the reference exposes is produced
by ``ft_build_tree`` bit-identically (as int32 on the device; ``.host()`` gives int64 numpy
views for comparison).

Beyond the reference fields each tree carries its ROWS: the unsplit root slices
(``row_fiber_ptr``, ``row_coord``).  The exact row-owner sweep of mode u walks tree u row by
row: root slice i of tree u is precisely the list of updates row i of A_u receives, in the
reference's serial order.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from .coo import as_device
from .errors import BuildError, ConfigError

DEFAULT_FIBER_THRESHOLD = 128
CORE_SEGMENT = 512  # max leaves per core-sweep row segment
LEAF_INDEX_MAX_ORDER = 6  # orders with the per-leaf prefix coordinates (the quad kernels)


@dataclass
class CsfTree:
    root_mode: int
    level_modes: tuple
    dims: tuple
    inds: tuple          # device int32, per depth
    ptrs: tuple          # device int32, per depth < N-1
    vals: object         # device fp32 [nnz]
    fiber_ptr: object    # device int32 [F+1]
    fiber_coord: object  # device int32 [F, N-1]
    sub_fiber_ptr: object
    sub_leaf_ptr: object
    row_fiber_ptr: object  # device int32 [rows+1]  (not a reference field)
    row_coord: object      # device int32 [rows]
    leaf_pc: object = None       # device int32 [nnz]  level-1 coordinate per leaf (derived)
    row_leaf_ptr: object = None  # device int32 [rows+1] first leaf per row (derived)
    seg_coord: object = None     # device int32 [segs]  core-sweep row segments (derived)
    seg_leaf_ptr: object = None  # device int32 [segs+1]
    slot_kb: int = 1             # leaves per row slot and batch (1 or 8)
    nfib: int = -1               # fiber count kept after drop_fibers()
    slot_grid: int = -1          # slot layout of the tcgen05 factor sweep (-1 = not planned,
    slot_batch_ptr: object = None  # 0 = does not apply); device int32 [G+1]
    slot_lc: object = None       # device int32 [batches x 128]
    slot_pc: object = None       # device int32 [batches x (N-2) x 128]
    slot_x: object = None        # device fp32 [batches x 128]
    _view: object = field(default=None, repr=False)
    num_subtensors_built: int = -1

    @property
    def order(self) -> int:
        return len(self.level_modes)

    @property
    def nnz(self) -> int:
        return int(self.vals.shape[0])

    @property
    def num_fibers(self) -> int:
        if self.nfib >= 0:
            return self.nfib
        return int(self.fiber_ptr.shape[0]) - 1

    def drop_fibers(self) -> "CsfTree":
        """Free fiber_ptr / fiber_coord (16 B per leaf at order 4) once the leaf-major index
        exists: the row-owner kernels (K3c, quadr, K4 quad, K6b) and the derived build of the next
        tree read leaf_pc / row_leaf_ptr / segments instead.  The fiber-walking kernels (hogwild
        K3a, dual / ws / gram, the uncached plan's counts) then refuse the tree.  What lets the
        BASELINE order-4 1 B-entry tensor's four trees fit one 180 GB GPU."""
        import torch

        if self.leaf_pc is None or self.row_leaf_ptr is None or self.seg_coord is None:
            raise ValueError("drop_fibers needs the leaf-major index and row segments")
        self.nfib = self.num_fibers
        empty = torch.empty(0, dtype=torch.int32, device=self.vals.device)
        self.fiber_ptr, self.fiber_coord = empty, empty
        self._view = None
        return self

    @property
    def num_subtensors(self) -> int:
        if self.num_subtensors_built >= 0:
            return self.num_subtensors_built
        return int(self.sub_fiber_ptr.shape[0]) - 1

    @property
    def num_rows(self) -> int:
        return int(self.row_coord.shape[0])

    @property
    def leaf_coord(self):
        return self.inds[-1]

    @property
    def prefix_modes(self) -> np.ndarray:
        return np.asarray(self.level_modes[:-1], dtype=np.int64)

    @property
    def leaf_mode(self) -> int:
        return self.level_modes[-1]

    def view(self) -> _lib.FtTree:
        """The ft_tree_t the kernels read (cached; arrays are kept alive by this object)."""
        if self._view is None:
            v = _lib.FtTree()
            v.order = self.order
            v.root_mode = self.root_mode
            v.nnz = self.nnz
            v.num_fibers = self.num_fibers
            v.num_rows = self.num_rows
            v.leaf_coord = self.leaf_coord.data_ptr()
            v.vals = self.vals.data_ptr()
            v.fiber_ptr = self.fiber_ptr.data_ptr() if self.nfib < 0 else None
            v.fiber_coord = self.fiber_coord.data_ptr() if self.nfib < 0 else None
            v.row_fiber_ptr = self.row_fiber_ptr.data_ptr()
            v.row_coord = self.row_coord.data_ptr()
            v.leaf_pc = _lib.ptr(self.leaf_pc)
            v.row_leaf_ptr = _lib.ptr(self.row_leaf_ptr)
            v.num_segs = 0 if self.seg_coord is None else int(self.seg_coord.shape[0])
            v.seg_coord = _lib.ptr(self.seg_coord)
            v.seg_leaf_ptr = _lib.ptr(self.seg_leaf_ptr)
            v.slot_grid = max(self.slot_grid, 0) if self.slot_lc is not None else 0
            v.slot_kb = self.slot_kb
            v.slot_batch_ptr = _lib.ptr(self.slot_batch_ptr)
            v.slot_lc = _lib.ptr(self.slot_lc)
            v.slot_pc = _lib.ptr(self.slot_pc)
            v.slot_x = _lib.ptr(self.slot_x)
            self._view = v
        return self._view

    def ensure_slots(self, J: int, R: int, stream=None) -> "CsfTree":
        """Build (once) the slot layout the tcgen05 factor sweep reads (K1d, ft_tree_slot_plan /
        ft_tree_slot_fill): the leaves re-ordered [CTA][batch][slot] so that each batch's
        coordinates and values are coalesced loads.  No-op when the sweep does not apply to this
        tree (too few rows to fill the GPU, J / R / order outside its cover, no leaf index)."""
        import torch

        if self.slot_grid >= 0 or self.row_leaf_ptr is None or self.leaf_pc is None:
            return self
        L = _lib.lib()
        g = ctypes.c_int32(0)
        kb = ctypes.c_int32(0)
        n = ctypes.c_int64(0)
        v = self.view()
        _lib.check(L.ft_tree_slot_plan(ctypes.byref(v), int(J), int(R), ctypes.byref(g),
                                       ctypes.byref(kb), None, ctypes.byref(n),
                                       _lib.stream_handle(stream)), "ft_tree_slot_plan")
        if g.value <= 0:
            self.slot_grid = 0
            return self
        i32 = dict(dtype=torch.int32, device=self.vals.device)
        bp = torch.empty(g.value + 1, **i32)
        _lib.check(L.ft_tree_slot_plan(ctypes.byref(v), int(J), int(R), ctypes.byref(g),
                                       ctypes.byref(kb), bp.data_ptr(), ctypes.byref(n),
                                       _lib.stream_handle(stream)), "ft_tree_slot_plan")
        length = int(n.value)
        lc = torch.empty(length, **i32)
        pc = torch.empty(length * (self.order - 2), **i32)
        x = torch.empty(length, dtype=torch.float32, device=self.vals.device)
        _lib.check(L.ft_tree_slot_fill(ctypes.byref(v), g.value, bp.data_ptr(), lc.data_ptr(),
                                       pc.data_ptr(), x.data_ptr(), _lib.stream_handle(stream)),
                   "ft_tree_slot_fill")
        self.slot_batch_ptr, self.slot_lc, self.slot_pc, self.slot_x = bp, lc, pc, x
        self.slot_grid = g.value
        self.slot_kb = kb.value
        self._view = None
        return self

    def host(self) -> dict:
        """All reference fields as int64 / float64 numpy arrays (for parity checks)."""
        c = lambda t: t.cpu().numpy().astype(np.int64)  # noqa: E731
        return {
            "inds": [c(a) for a in self.inds],
            "ptrs": [c(a) for a in self.ptrs],
            "vals": self.vals.cpu().numpy().astype(np.float64),
            "fiber_ptr": c(self.fiber_ptr),
            "fiber_coord": c(self.fiber_coord),
            "sub_fiber_ptr": c(self.sub_fiber_ptr),
            "sub_leaf_ptr": c(self.sub_leaf_ptr),
            "row_fiber_ptr": c(self.row_fiber_ptr),
            "row_coord": c(self.row_coord),
        }

    def slice_rows(self, r0: int, r1: int) -> "CsfTree":
        """A compact copy holding only root slices [r0, r1) (multi-GPU row blocks), with the
        fiber / leaf pointers rebased.  Subtensor and per-depth arrays are not sliced (the sweep
        kernels do not read them); they are left empty."""
        import torch

        f0 = int(self.row_fiber_ptr[r0])
        f1 = int(self.row_fiber_ptr[r1])
        l0 = int(self.fiber_ptr[f0])
        l1 = int(self.fiber_ptr[f1])
        empty = torch.empty(0, dtype=torch.int32, device=self.vals.device)
        inds = tuple(empty for _ in range(self.order - 1)) + (self.leaf_coord[l0:l1].clone(),)
        out = CsfTree(
            root_mode=self.root_mode, level_modes=self.level_modes, dims=self.dims,
            inds=inds, ptrs=tuple(empty for _ in self.ptrs),
            vals=self.vals[l0:l1].clone(),
            fiber_ptr=(self.fiber_ptr[f0:f1 + 1] - l0).contiguous(),
            fiber_coord=self.fiber_coord[f0:f1].clone(),
            sub_fiber_ptr=torch.zeros(1, dtype=torch.int32, device=self.vals.device),
            sub_leaf_ptr=torch.zeros(1, dtype=torch.int32, device=self.vals.device),
            row_fiber_ptr=(self.row_fiber_ptr[r0:r1 + 1] - f0).contiguous(),
            row_coord=self.row_coord[r0:r1].clone(),
            leaf_pc=None if self.leaf_pc is None else self.leaf_pc[l0:l1].clone(),
            row_leaf_ptr=None if self.row_leaf_ptr is None
            else (self.row_leaf_ptr[r0:r1 + 1] - l0).contiguous(),
        )
        return out if out.row_leaf_ptr is None or out.num_rows == 0 else add_row_segments(out)


@dataclass
class CsfForest:
    """One tree per root mode over the same entry multiset (csf.py:83-88)."""

    trees: tuple
    fiber_threshold: object
    omega: int | None = None   # |Omega| of the whole tensor when trees hold a row-block shard


def _trim(buf, n):
    """First n entries of a capacity buffer: a view when that keeps most of it (no transient
    copy of a multi-GB array), a compact copy otherwise."""
    return buf[:n] if n >= 0.75 * buf.numel() else buf[:n].clone()


def build_tree(tensor, root_mode: int, fiber_threshold=DEFAULT_FIBER_THRESHOLD,
               stream=None, compact: bool = False, keep_fibers: bool = True) -> CsfTree:
    """GPU B-CSF build (csf.py:101-196).  ``tensor``: SparseCooTensor or DeviceCoo.

    ``compact=True`` keeps only what the sweep kernels read (leaf coordinates, values,
    fiber_ptr / fiber_coord, rows): the per-depth ``inds`` / ``ptrs`` and the subtensor arrays
    -- reference-format fields -- are not built (saves ~40 % of a tree at order 4).
    ``keep_fibers=False`` (compact only) does not build fiber_coord at all and drops fiber_ptr
    once the leaf-major index exists (CsfTree.drop_fibers)."""
    import torch

    L = _lib.lib()
    dev = as_device(tensor)
    N, nnz = dev.order, dev.nnz
    if nnz == 0:
        raise BuildError("cannot index an empty tensor")
    if not 0 <= root_mode < N:
        raise ConfigError(f"root_mode must be in [0, {N}), got {root_mode}")
    if fiber_threshold is None:
        thr = 0
    else:
        thr = int(fiber_threshold)
        if thr < 1:
            raise ConfigError(f"fiber_threshold must be >= 1, got {fiber_threshold}")
    dims = tuple(dev.dims)

    def call(out):
        return L.ft_build_tree(N, nnz, out["dims"], dev.idx.data_ptr(), dev.vals.data_ptr(),
                               root_mode, thr, *out["args"])

    def on_duplicate(counts):
        e = int(counts[3])
        coord = dev.idx[e].cpu().numpy()
        from .errors import ValidationError

        raise ValidationError(f"duplicate coordinate {tuple(int(c) + 1 for c in coord)}")

    return _build_with(call, N, nnz, dims, root_mode, compact, stream, "ft_build_tree",
                       on_duplicate, keep_fibers)


def build_tree_derived(prev: CsfTree, fiber_threshold=DEFAULT_FIBER_THRESHOLD, stream=None,
                       compact: bool = False, keep_fibers: bool = True):
    """The tree rooted at ``prev.root_mode + 1`` from ``prev``'s leaf order (K1 derived build,
    ``ft_build_tree_derived``): a stable radix sort on a 32-bit key instead of the full-width
    COO sort; bit-identical to ``build_tree``.  None when it does not apply (prev without the
    leaf-major index, or a key wider than 32 bits)."""
    if prev.leaf_pc is None or prev.row_leaf_ptr is None:
        return None
    L = _lib.lib()
    N, nnz = prev.order, prev.nnz
    dims = tuple(prev.dims)
    thr = 0 if fiber_threshold is None else int(fiber_threshold)
    root_mode = (prev.root_mode + 1) % N
    pv = prev.view()

    def call(out):
        return L.ft_build_tree_derived(ctypes.byref(pv), out["dims"], thr, *out["args"])

    try:
        return _build_with(call, N, nnz, dims, root_mode, compact, stream,
                           "ft_build_tree_derived", None, keep_fibers)
    except _Unsupported:
        return None


class _Unsupported(Exception):
    pass


def _build_with(call, N, nnz, dims, root_mode, compact, stream, what, on_duplicate,
                keep_fibers=True):
    """Allocate a build's output buffers, run ``call`` (an ft_build_tree* entry point), trim and
    wrap them as a CsfTree with its leaf-major index."""
    import torch

    i32 = dict(dtype=torch.int32, device="cuda")
    leaf_vals = torch.empty(nnz, dtype=torch.float32, device="cuda")
    leaf = torch.empty(nnz, **i32)
    inds = [torch.empty(nnz, **i32) for _ in range(N - 1)] + [leaf] if not compact else [leaf]
    ptrs = [torch.empty(nnz + 1, **i32) for _ in range(N - 1)] if not compact else []
    fiber_ptr = torch.empty(nnz + 1, **i32)
    no_coord = compact and not keep_fibers and 3 <= N <= _leaf_index_max_order()
    fiber_coord = None if no_coord else torch.empty(nnz * (N - 1), **i32)
    sub_fiber_ptr = torch.empty(nnz + 1, **i32) if not compact else None
    sub_leaf_ptr = torch.empty(nnz + 1, **i32) if not compact else None
    row_fiber_ptr = torch.empty(nnz + 1, **i32)
    row_coord = torch.empty(nnz, **i32)
    counts = np.zeros(4 + N, dtype=np.int64)
    leaf_pc = torch.empty((nnz, N - 2), **i32) if 3 <= N <= _leaf_index_max_order() else None
    ind_ptrs = [None] * (N - 1) + [leaf.data_ptr()] if compact else [a.data_ptr() for a in inds]
    ind_tab = (ctypes.c_void_p * N)(*ind_ptrs)
    ptr_tab = None if compact else (ctypes.c_void_p * max(N - 1, 1))(*[a.data_ptr() for a in ptrs])
    out = {"dims": (ctypes.c_int64 * N)(*dims),
           "args": (leaf_vals.data_ptr(), ind_tab, ptr_tab, fiber_ptr.data_ptr(),
                    _lib.ptr(fiber_coord), _lib.ptr(sub_fiber_ptr), _lib.ptr(sub_leaf_ptr),
                    row_fiber_ptr.data_ptr(), row_coord.data_ptr(),
                    counts.ctypes.data_as(ctypes.POINTER(ctypes.c_int64)), _lib.ptr(leaf_pc),
                    _lib.stream_handle(stream))}
    rc = call(out)
    if rc == _lib.FT_ERR_DUPLICATE and on_duplicate is not None:
        on_duplicate(counts)
    if rc == _lib.FT_ERR_UNSUPPORTED and on_duplicate is None:
        raise _Unsupported(what)
    _lib.check(rc, what)
    F, S, rows = int(counts[0]), int(counts[1]), int(counts[2])
    nodes = [int(c) for c in counts[4:4 + N]]
    empty = torch.empty(0, **i32)
    if compact:
        inds_t = tuple(empty for _ in range(N - 1)) + (leaf,)
        ptrs_t = tuple(empty for _ in range(N - 1))
        sfp = slp = torch.zeros(1, **i32)
    else:
        inds_t = tuple(_trim(inds[d], nodes[d]) for d in range(N))
        ptrs_t = tuple(_trim(ptrs[d], nodes[d] + 1) for d in range(N - 1))
        sfp, slp = _trim(sub_fiber_ptr, S + 1), _trim(sub_leaf_ptr, S + 1)
    tree = CsfTree(
        root_mode=root_mode,
        level_modes=tuple((root_mode + d) % N for d in range(N)),
        dims=tuple(dims),
        inds=inds_t,
        ptrs=ptrs_t,
        vals=leaf_vals,
        fiber_ptr=_trim(fiber_ptr, F + 1),
        fiber_coord=(torch.empty((0, N - 1), **i32) if fiber_coord is None
                     else _trim(fiber_coord, F * (N - 1)).view(F, N - 1)),
        sub_fiber_ptr=sfp,
        sub_leaf_ptr=slp,
        row_fiber_ptr=_trim(row_fiber_ptr, rows + 1),
        row_coord=_trim(row_coord, rows),
    )
    tree.num_subtensors_built = S
    add_leaf_index(tree, stream, leaf_pc=leaf_pc)
    if no_coord:
        tree.drop_fibers()
    return tree


def _leaf_index_max_order() -> int:
    import os

    return min(int(os.environ.get("FT_LEAF_INDEX_MAX_ORDER", LEAF_INDEX_MAX_ORDER)), 6)


def add_leaf_index(tree: CsfTree, stream=None, leaf_pc=None) -> CsfTree:
    """Derive the leaf-major index the row-owner kernels read (K1b, ft_tree_leaf_index):
    ``leaf_pc`` (each leaf's prefix coordinates, levels 1..N-2, for orders 3-6) and
    ``row_leaf_ptr`` (first leaf of each root slice).  Not reference fields."""
    import torch

    i32 = dict(dtype=torch.int32, device=tree.vals.device)
    N = tree.order
    # prefix levels per leaf (4 (N-2) bytes per leaf) up to LEAF_INDEX_MAX_ORDER.  The K4 core
    # (direct register loads) uses them at every order (order-6 10K^6: 15.2 -> 8.3 ms per
    # mode); the factor sweep's quad fold pays at orders 3-4 only (order 6: 30.6 vs 24.2 ms
    # dual), so orders 5-6 keep the fiber-walking factor kernels (sweep.cu auto dispatch)
    have = leaf_pc is not None  # already written by the build (from its sorted level columns)
    tree.leaf_pc = leaf_pc if have else (
        torch.empty((tree.nnz, N - 2), **i32) if 3 <= N <= _leaf_index_max_order() else None)
    tree.row_leaf_ptr = torch.empty(tree.num_rows + 1, **i32)
    tree._view = None
    v = tree.view()
    _lib.check(_lib.lib().ft_tree_leaf_index(ctypes.byref(v),
                                             None if have else _lib.ptr(tree.leaf_pc),
                                             tree.row_leaf_ptr.data_ptr(),
                                             _lib.stream_handle(stream)), "ft_tree_leaf_index")
    tree._view = None
    return add_row_segments(tree, stream)


def add_row_segments(tree: CsfTree, stream=None) -> CsfTree:
    """Core-sweep row segments (K1c, ft_tree_row_segments): rows cut at CORE_SEGMENT leaves so
    few long rows still fill the GPU in the core sweep (a sum over each row's leaves, so the
    pieces are independent).  Needs ``row_leaf_ptr``."""
    import torch

    i32 = dict(dtype=torch.int32, device=tree.vals.device)
    tree._view = None
    rows = tree.num_rows
    cap = rows + tree.nnz // CORE_SEGMENT + 1
    seg_coord = torch.empty(cap, **i32)
    seg_ptr = torch.empty(cap + 1, **i32)
    nseg = np.zeros(1, dtype=np.int64)
    _lib.check(_lib.lib().ft_tree_row_segments(
        ctypes.byref(tree.view()), CORE_SEGMENT, seg_coord.data_ptr(), seg_ptr.data_ptr(),
        nseg.ctypes.data_as(ctypes.POINTER(ctypes.c_int64)), _lib.stream_handle(stream)),
        "ft_tree_row_segments")
    n = int(nseg[0])
    tree.seg_coord = _trim(seg_coord, n)
    tree.seg_leaf_ptr = _trim(seg_ptr, n + 1)
    tree._view = None
    return tree


def build_forest(tensor, fiber_threshold=DEFAULT_FIBER_THRESHOLD, stream=None,
                 compact: bool = False, concurrent: bool = False,
                 derived: bool = True, keep_fibers: bool = True) -> CsfForest:
    """All N trees (csf.py:199-201).  ``concurrent=True`` builds each tree on its own CUDA
    stream from its own host thread (ctypes releases the GIL); the result is identical, but it
    measured slower (Netflix: 33 ms vs 26.5 ms sequential, with 100-200 ms outliers while the
    per-stream allocator pools grow), so it is off by default."""
    import torch

    dev = as_device(tensor)
    N = dev.order
    if not concurrent or N == 1:
        # tree 0 from the COO, tree t from tree t-1's leaf order when the 32-bit derived sort
        # applies (bit-identical; Netflix: 4 radix passes of 4-byte keys instead of 6 of 8-byte)
        # keep_fibers=False: each tree's fiber arrays are freed as soon as the next tree is
        # derived from it (tree t+1's build reads only tree t's leaf-major index)
        # (compact builds without fibers never compute fiber_coord at all)
        kf = keep_fibers or not compact
        trees = [build_tree(dev, 0, fiber_threshold, stream, compact, kf)]
        for t in range(1, N):
            tree = build_tree_derived(trees[-1], fiber_threshold, stream, compact, kf) \
                if derived else None
            if not keep_fibers and trees[-1].nfib < 0:
                trees[-1].drop_fibers()
            trees.append(tree if tree is not None
                         else build_tree(dev, t, fiber_threshold, stream, compact, kf))
        if not keep_fibers and trees[-1].nfib < 0:
            trees[-1].drop_fibers()
        return CsfForest(trees=tuple(trees), fiber_threshold=fiber_threshold)
    from concurrent.futures import ThreadPoolExecutor

    main = stream if stream is not None else torch.cuda.current_stream()
    device = torch.cuda.current_device()
    streams = [torch.cuda.Stream(device=device) for _ in range(N)]
    for s in streams:
        s.wait_stream(main)  # the COO is ready on the caller's stream

    def one(t):
        torch.cuda.set_device(device)  # worker threads start on device 0
        with torch.cuda.stream(streams[t]):
            return build_tree(dev, t, fiber_threshold, streams[t], compact)

    with ThreadPoolExecutor(max_workers=N) as ex:
        trees = tuple(ex.map(one, range(N)))
    for s, tree in zip(streams, trees):
        main.wait_stream(s)
        # the caller's stream uses (and later frees) these buffers: tell the allocator
        for name in ("vals", "fiber_ptr", "fiber_coord", "sub_fiber_ptr", "sub_leaf_ptr",
                     "row_fiber_ptr", "row_coord", "leaf_pc", "row_leaf_ptr", "seg_coord",
                     "seg_leaf_ptr"):
            a = getattr(tree, name)
            if a is not None:
                a.record_stream(main)
        for a in tuple(tree.inds) + tuple(tree.ptrs):
            a.record_stream(main)
    return CsfForest(trees=trees, fiber_threshold=fiber_threshold)
