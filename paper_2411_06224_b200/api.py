"""The reference's hot-path interface (adipc/sparse, adipc/precond,
adipc/solver/pcg.hpp), same names, argument meaning and error behaviour,
executed on the B200 through the C-ABI. Host-side data containers mirror the
reference structs; the numeric work runs in libadipc_gpu.so.

  reference                                            here
  sparse/block_coo.hpp:13-21   make_block_key ...      make_block_key, block_key_row, block_key_col
  sparse/block_coo.hpp:25-51   BlockTripletStream      BlockTripletStream (keys u64[T], values f64[T,9] col-major)
  sparse/block_coo.hpp:54-61   SortedSymBlockCoo       SortedSymBlockCoo
  sparse/block_coo.hpp:106     sort_stream             sort_stream (GPU)
  sparse/reduction.hpp:30      fast_segment_reduction  fast_segment_reduction (GPU)
  sparse/reduction.hpp:83      fast_hash_reduction     fast_hash_reduction (GPU)
  sparse/srbk_spmv.hpp:13      srbk_spmv               srbk_spmv (GPU)
  sparse/srbk_spmv.hpp:52      dump_block_coo          dump_block_coo
  sparse/block_split.hpp       split_*                 split_12x12, split_sym_12x12, split_12x3, split_3x12
  sparse/abd_reduce.hpp        DofMap, two_level_...   DofMap, two_level_abd_reduce (GPU)
  precond/partition.hpp        subdomain_count, Partition, chunk_partition, partition_block_graph (native host)
  precond/hierarchy.hpp        MasHierarchy, build_hierarchy (native host)
  precond/mas.hpp              Preconditioner, block_edges, MasPreconditioner (GPU)
  precond/block_jacobi.hpp     BlockJacobiPreconditioner (GPU)
  solver/pcg.hpp               PcgResult, pcg_solve (GPU)
"""
from __future__ import annotations

import ctypes as C

import numpy as np

from . import _lib
from ._lib import ptr
from .context import Context, IndefiniteSubdomain, InvalidArgument, PcgResult, default_context

__all__ = [
    "ExecPolicy", "make_block_key", "block_key_row", "block_key_col", "BlockTripletStream", "SortedSymBlockCoo",
    "sort_stream", "fast_segment_reduction", "fast_hash_reduction", "srbk_spmv", "dump_block_coo", "load_matrix_binary", "split_12x12",
    "split_sym_12x12", "split_12x3", "split_3x12", "DofMap", "two_level_abd_reduce", "subdomain_count", "Partition",
    "chunk_partition", "partition_block_graph", "MasHierarchy", "build_hierarchy", "block_edges", "Preconditioner",
    "MasPreconditioner", "BlockJacobiPreconditioner", "PcgResult", "pcg_solve", "IndefiniteSubdomain",
    "InvalidArgument",
]


class ExecPolicy:
    """core/parallel.hpp:18-22. On the GPU `threads`/`lane_width` have no
    effect (a warp is the lane group); results always equal the reference's
    deterministic mode for the reductions."""

    def __init__(self, deterministic: bool = False, threads: int = 0, lane_width: int = 32, device: int = 0):
        self.deterministic = deterministic
        self.threads = threads
        self.lane_width = lane_width
        self.device = device


def _ctx(pol) -> Context:
    return default_context(pol.device if pol is not None else 0)


def make_block_key(row: int, col: int) -> int:
    return (int(row) << 32) | int(col)


def block_key_row(k: int) -> int:
    return int(k) >> 32


def block_key_col(k: int) -> int:
    return int(k) & 0xFFFFFFFF


class BlockTripletStream:
    """block_coo.hpp:25-51: keys u64[T], values f64[T, 9] (Mat3 column-major)."""

    def __init__(self, keys=None, values=None):
        self._k = [] if keys is None else list(np.asarray(keys, np.uint64))
        self._v = [] if values is None else list(np.asarray(values, np.float64).reshape(-1, 9))
        self._arr = None

    def emit(self, r: int, c: int, m):
        """m: natural 3x3 array. Below-diagonal blocks are stored transposed."""
        m = np.asarray(m, np.float64).reshape(3, 3)
        if r <= c:
            self._k.append(np.uint64(make_block_key(r, c)))
            self._v.append(np.ascontiguousarray(m.T).reshape(-1))
        else:
            self._k.append(np.uint64(make_block_key(c, r)))
            self._v.append(np.ascontiguousarray(m).reshape(-1))
        self._arr = None

    def append(self, other: "BlockTripletStream"):
        self._k.extend(other.keys)
        self._v.extend(other.values)
        self._arr = None

    def _arrays(self):
        if self._arr is None:
            k = np.array(self._k, np.uint64) if self._k else np.zeros(0, np.uint64)
            v = np.array(self._v, np.float64).reshape(-1, 9) if self._v else np.zeros((0, 9))
            self._arr = (k, v)
        return self._arr

    @property
    def keys(self):
        return self._arrays()[0]

    @property
    def values(self):
        return self._arrays()[1]

    def set(self, keys, values):
        self._k = list(keys)
        self._v = list(values)
        self._arr = (np.asarray(keys, np.uint64), np.asarray(values, np.float64).reshape(-1, 9))

    def size(self):
        return len(self._k)

    def clear(self):
        self._k, self._v, self._arr = [], [], None


class SortedSymBlockCoo:
    """block_coo.hpp:54-61."""

    def __init__(self, n_block_rows=0, rows=None, cols=None, blocks=None):
        self.n_block_rows = n_block_rows
        self.rows = np.zeros(0, np.uint32) if rows is None else np.asarray(rows, np.uint32)
        self.cols = np.zeros(0, np.uint32) if cols is None else np.asarray(cols, np.uint32)
        self.blocks = np.zeros((0, 9)) if blocks is None else np.asarray(blocks, np.float64).reshape(-1, 9)

    def size(self):
        return len(self.blocks)


def sort_stream(s: BlockTripletStream, pol: ExecPolicy | None = None) -> None:
    """block_coo.hpp:106-113, in place, stable."""
    if s.size() == 0:
        return
    k, v = _ctx(pol).sort_stream(s.keys, s.values)
    s.set(k, v)


def fast_segment_reduction(O, values, n_segments: int, pol: ExecPolicy | None = None):
    """reduction.hpp:30-79 for V = Real ([n]), Vec3 ([n,3]) or Mat3 ([n,9])."""
    V = np.asarray(values, np.float64)
    if len(O) != V.shape[0]:
        raise InvalidArgument("segment map size mismatch")
    return _ctx(pol).segment_reduce(O, V, n_segments)


def fast_hash_reduction(sorted_stream: BlockTripletStream, n_block_rows: int,
                        pol: ExecPolicy | None = None) -> SortedSymBlockCoo:
    """reduction.hpp:83-107."""
    if sorted_stream.size() == 0:
        return SortedSymBlockCoo(n_block_rows)
    ctx = _ctx(pol)
    ctx.assemble(sorted_stream.keys, sorted_stream.values, n_block_rows, deterministic=True)
    n, rows, cols, blocks = ctx.copy_matrix()
    return SortedSymBlockCoo(n_block_rows, rows, cols, blocks)


def srbk_spmv(A: SortedSymBlockCoo, x, pol: ExecPolicy | None = None):
    """srbk_spmv.hpp:13-49: y = A x over the upper-stored blocks. x: [n,3] or [3n]."""
    xa = np.asarray(x, np.float64)
    shape = xa.shape
    if A.size() == 0:
        return np.zeros(shape)
    ctx = _ctx(pol)
    ctx.set_matrix(A.n_block_rows, A.rows, A.cols, A.blocks)
    return ctx.spmv(xa.reshape(-1)).reshape(shape)


def dump_block_coo(A: SortedSymBlockCoo, f) -> None:
    """srbk_spmv.hpp:52-60: 'n U' header, then 'row col' + the 9 values
    row-major per block, each as a default-formatted C++ ostream double
    (printf %g: 6 significant digits) — byte-identical to the reference's
    --dump-hessian text."""
    f.write(f"{A.n_block_rows} {A.size()}\n")
    for r, c, b in zip(A.rows, A.cols, A.blocks):
        nat = np.asarray(b, np.float64).reshape(3, 3).T  # column-major storage -> row-major
        f.write(f"{int(r)} {int(c)} " + " ".join("%g" % float(v) for v in nat.reshape(-1)) + "\n")


def load_matrix_binary(path) -> SortedSymBlockCoo:
    """Reads adipc_gpu_dump_matrix_binary's capture ("ADIPCMAT", version 1)."""
    with open(path, "rb") as f:
        head = f.read(24)
        if len(head) != 24 or head[:8] != b"ADIPCMAT":
            raise ValueError("not an ADIPCMAT capture")
        version, n = np.frombuffer(head[8:16], np.uint32)[0], int(np.frombuffer(head[12:16], np.int32)[0])
        if version != 1:
            raise ValueError(f"unsupported ADIPCMAT version {version}")
        U = int(np.frombuffer(head[16:24], np.int64)[0])
        rows = np.frombuffer(f.read(4 * U), np.uint32).copy()
        cols = np.frombuffer(f.read(4 * U), np.uint32).copy()
        blocks = np.frombuffer(f.read(72 * U), np.float64).reshape(U, 9).copy()
    return SortedSymBlockCoo(n, rows, cols, blocks)


# -- block_split.hpp:10-33 (host tiling helpers used by producers) -----------
def split_12x12(row_base, col_base, H, out: BlockTripletStream):
    H = np.asarray(H, np.float64)
    for ti in range(4):
        for tj in range(4):
            out.emit(row_base + ti, col_base + tj, H[3 * ti:3 * ti + 3, 3 * tj:3 * tj + 3])


def split_sym_12x12(base, H, out: BlockTripletStream):
    H = np.asarray(H, np.float64)
    for ti in range(4):
        for tj in range(ti, 4):
            out.emit(base + ti, base + tj, H[3 * ti:3 * ti + 3, 3 * tj:3 * tj + 3])


def split_12x3(row_base, col, H, out: BlockTripletStream):
    H = np.asarray(H, np.float64)
    for t in range(4):
        out.emit(row_base + t, col, H[3 * t:3 * t + 3, :])


def split_3x12(row, col_base, H, out: BlockTripletStream):
    H = np.asarray(H, np.float64)
    for t in range(4):
        out.emit(row, col_base + t, H[:, 3 * t:3 * t + 3])


class DofMap:
    """abd_reduce.hpp:11-27. abd_node_jacobian: list/array of 3x12 (natural)."""

    def __init__(self, n_fem_nodes=0, n_bodies=0, abd_node_body=None, abd_node_jacobian=None):
        self.n_fem_nodes = n_fem_nodes
        self.n_bodies = n_bodies
        self.abd_node_body = [] if abd_node_body is None else list(abd_node_body)
        self.abd_node_jacobian = [] if abd_node_jacobian is None else list(abd_node_jacobian)

    def n_nodes(self):
        return self.n_fem_nodes + len(self.abd_node_body)

    def n_blocks(self):
        return self.n_fem_nodes + 4 * self.n_bodies

    def jac36(self):
        if not self.abd_node_jacobian:
            return np.zeros((0, 36))
        return np.array([np.ascontiguousarray(np.asarray(J, np.float64).T).reshape(-1)
                         for J in self.abd_node_jacobian])


def two_level_abd_reduce(node_pairs: BlockTripletStream, dof_map: DofMap,
                         pol: ExecPolicy | None = None) -> BlockTripletStream:
    """abd_reduce.hpp:32-74: level-1 sort+reduce of node-pair blocks, then
    J^T C J tiles in the reference's order."""
    if node_pairs.size() == 0:
        return BlockTripletStream()
    k, v = _ctx(pol).two_level_abd_reduce(node_pairs.keys, node_pairs.values, dof_map.n_fem_nodes,
                                          dof_map.n_bodies, dof_map.abd_node_body, dof_map.jac36())
    out = BlockTripletStream()
    out.set(k, v)
    return out


# -- precond/partition.hpp -------------------------------------------------------
class Partition:
    def __init__(self, part_of=None, n_parts=0, capacity=0):
        self.part_of = np.zeros(0, np.int32) if part_of is None else np.asarray(part_of, np.int32)
        self.n_parts = n_parts
        self.capacity = capacity


def subdomain_count(v, n, n_o):
    return _lib.gpu().adipc_subdomain_count(v, n, n_o)


def chunk_partition(v, capacity) -> Partition:
    part = np.empty(max(v, 1), np.int32)
    n = _lib.gpu().adipc_chunk_partition(v, capacity, ptr(part))
    return Partition(part[:v].copy(), n, capacity)


def _edge_array(edges):
    e = np.ascontiguousarray(np.asarray(edges, np.int32).reshape(-1, 2))
    return e, len(e)


def partition_block_graph(v, edges, capacity) -> Partition:
    e, ne = _edge_array(edges)
    part = np.empty(max(v, 1), np.int32)
    n = _lib.gpu().adipc_partition_block_graph(v, ptr(e), ne, capacity, ptr(part))
    return Partition(part[:v].copy(), n, capacity)


class MasHierarchy:
    """hierarchy.hpp:15-28; `levels` are dicts n_nodes / n_parts / part_of / agg."""

    def __init__(self, handle, n_slots, capacity):
        self.h = handle
        self.n_slots = n_slots
        self.capacity = capacity
        L = _lib.gpu()
        self.levels = []
        for l in range(L.adipc_hierarchy_n_levels(handle)):
            nn, npart = C.c_int32(), C.c_int32()
            L.adipc_hierarchy_level(handle, l, C.byref(nn), C.byref(npart), None, None)
            part = np.empty(nn.value, np.int32)
            agg = np.empty(n_slots, np.int32)
            L.adipc_hierarchy_level(handle, l, C.byref(nn), C.byref(npart), ptr(part), ptr(agg))
            self.levels.append(dict(n_nodes=nn.value, n_parts=npart.value, part_of=part, agg=agg))

    def n_levels(self):
        return len(self.levels)

    def __del__(self):
        if getattr(self, "h", None):
            _lib.gpu().adipc_hierarchy_free(self.h)
            self.h = None


def build_hierarchy(l0: Partition, edges, max_levels: int) -> MasHierarchy:
    e, ne = _edge_array(edges)
    p = np.ascontiguousarray(l0.part_of, np.int32)
    h = _lib.gpu().adipc_build_hierarchy(ptr(p), len(p), l0.n_parts, l0.capacity, ptr(e), ne, max_levels)
    return MasHierarchy(C.c_void_p(h), len(p), l0.capacity)


def block_edges(A: SortedSymBlockCoo):
    """mas.hpp:19-25."""
    m = A.rows != A.cols
    return np.stack([A.rows[m].astype(np.int32), A.cols[m].astype(np.int32)], axis=1)


# -- preconditioners --------------------------------------------------------------
class Preconditioner:
    """mas.hpp:12-15: apply(r) -> z."""

    def __init__(self, device: int = 0):
        self.ctx = Context(device)
        self._A = None

    def _upload(self, A: SortedSymBlockCoo):
        self.ctx.set_matrix(A.n_block_rows, A.rows, A.cols, A.blocks)
        self._A = A

    def apply(self, r):
        return self.ctx.precond_apply(r)


class MasPreconditioner(Preconditioner):
    """mas.hpp:32-115 (build: Galerkin restriction + batched Cholesky inverse
    on the GPU; apply: per-level dense solves, summed)."""

    def build(self, A: SortedSymBlockCoo, h: MasHierarchy):
        self._upload(A)
        self.ctx.build_mas(h)
        self._n_levels = h.n_levels()

    def n_levels(self):
        return self._n_levels

    def level_inverse(self, l, s):
        return self.ctx.subdomain_inverse(l, s)


class BlockJacobiPreconditioner(Preconditioner):
    """block_jacobi.hpp:8-26."""

    def build(self, A: SortedSymBlockCoo):
        self._upload(A)
        self.ctx.build_preconditioner(_lib.PRECOND_JACOBI)


def pcg_solve(A: SortedSymBlockCoo, b, M: Preconditioner, rel_tol: float, restart: int, max_iters: int,
              pol: ExecPolicy | None = None):
    """pcg.hpp:34-88. Returns (x, PcgResult)."""
    if M._A is not A:
        raise InvalidArgument("pcg_solve: the preconditioner must be built on this matrix")
    return M.ctx.pcg(np.asarray(b, np.float64).reshape(-1), rel_tol, restart, max_iters)
