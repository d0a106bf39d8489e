"""Structural preprocessing in front of the Gray walk.

Same functions and semantics as permkit.preprocess
(/root/reference/pkg/src/permkit/preprocess.py):

* the matching filter -- Hopcroft-Karp maximum matching (:75-119), strongly
  connected components of the matched-pair digraph (:152-218), deletion of
  entries that lie on no perfect matching (:221-248);
* the compressions d1 / d2 / d34 of a sparsest row or column (:257-364);
* the decomposition driver decomp_run (:420-507): a LIFO worklist that
  compresses until every row and column has more than `min_nnz_threshold`
  nonzeros and then evaluates the leaf permanent.

What changes for the B200 is the leaf evaluation. permkit calls perm_nw /
perm_spa once per leaf (preprocess.py:495-504), which on a GPU would be one
tiny launch per leaf. Here kernel leaves are queued and evaluated in batches:
every (kind, order) group goes to ONE launch of the batched walk kernels
(pk_dense_f64_batch / pk_dense_c128_batch, permanent_batch); integer leaves
go to the exact integer kernels one matrix per call. Contributions are
combined exactly as permkit does -- sorted by task id, double-double
(:398-417) -- so the evaluation order never affects the result.

The worklist itself runs on a light row-list form of each task matrix (the
reference rebuilds a CRS/CCS pair per task); every value is computed with the
same Python scalar operations in the same order, so leaf matrices and
multipliers are identical to permkit's (tests/test_preprocess.py checks them
against the reference's own leaves).
"""

from __future__ import annotations

import time
from collections import defaultdict, deque
from dataclasses import dataclass, field
from typing import Dict, List, NamedTuple, Optional, Sequence, Tuple, Union

from .errors import DecompTimeout, StructureError
from .matrix import (KIND_COMPLEX, KIND_INT, Scalar, SparsePair, sparse_from_triplets)
from .precision import AccumulatorPolicy, DoubleDouble, as_policy, dd_add

DENSE_LEAF_DENSITY = 0.30
DEFAULT_TASK_LIMIT = 10_000_000
DEFAULT_TIME_LIMIT = 600.0
LEAF_BATCH = 4096  # kernel leaves queued before a batched evaluation

Rows = List[List[Tuple[int, Scalar]]]  # per row: (column, value), columns ascending


# ---------------------------------------------------------------------------
# bipartite matching and components


@dataclass(frozen=True)
class BipartiteGraph:
    """Rows vs columns, one edge per stored nonzero (preprocess.py:49-62)."""

    n: int
    row_adj: Tuple[Tuple[int, ...], ...]

    @classmethod
    def from_sparse(cls, s: SparsePair) -> "BipartiteGraph":
        crs = s.crs
        return cls(s.n, tuple(tuple(crs.cids[crs.rptrs[i]:crs.rptrs[i + 1]])
                              for i in range(s.n)))


@dataclass(frozen=True)
class Matching:
    row_to_col: Tuple[int, ...]  # -1 where unmatched
    col_to_row: Tuple[int, ...]
    size: int

    @property
    def perfect(self) -> bool:
        return self.size == len(self.row_to_col)


def max_matching(graph: BipartiteGraph) -> Matching:
    """Maximum bipartite matching by Hopcroft-Karp (preprocess.py:75-119):
    BFS layers from the free rows, then vertex-disjoint shortest augmenting
    paths found by an explicit-stack DFS; rows and edges in index order."""
    n, adj = graph.n, graph.row_adj
    r2c = [-1] * n
    c2r = [-1] * n
    size = 0
    while True:
        layer = [-1] * n
        q = deque(r for r in range(n) if r2c[r] == -1)
        for r in q:
            layer[r] = 0
        found = False
        while q:
            r = q.popleft()
            for c in adj[r]:
                r2 = c2r[c]
                if r2 == -1:
                    found = True
                elif layer[r2] == -1:
                    layer[r2] = layer[r] + 1
                    q.append(r2)
        if not found:
            break
        for root in range(n):
            if r2c[root] != -1:
                continue
            # DFS along layer + 1 edges; path = stack of (row, next edge index)
            path = [[root, 0]]
            while path:
                r, k = path[-1]
                if k == len(adj[r]):
                    layer[r] = -2  # dead end for this phase
                    path.pop()
                    continue
                path[-1][1] = k + 1
                c = adj[r][k]
                r2 = c2r[c]
                if r2 == -1:
                    # augment along the path
                    for rr, kk in reversed(path):
                        cc = adj[rr][kk - 1]
                        c2r[cc] = rr
                        r2c[rr] = cc
                    size += 1
                    break
                if layer[r2] == layer[r] + 1:
                    path.append([r2, 0])
    return Matching(tuple(r2c), tuple(c2r), size)


@dataclass(frozen=True)
class SccLabeling:
    count: int
    row_component: Tuple[int, ...]
    col_component: Tuple[int, ...]


@dataclass(frozen=True)
class SingularVerdict:
    """Structural certificate that the permanent is exactly zero."""

    reason: str

    @property
    def value(self) -> int:
        return 0


@dataclass(frozen=True)
class DmResult:
    matching: Matching
    labeling: SccLabeling
    removed: Tuple[Tuple[int, int], ...]
    filtered: SparsePair
    nnz_before: int
    nnz_after: int


def strongly_connected(adj: Sequence[Sequence[int]]) -> Tuple[int, List[int]]:
    """Tarjan's algorithm with an explicit stack; (count, node -> component)."""
    n = len(adj)
    order = [-1] * n
    low = [0] * n
    comp = [-1] * n
    onstack = [False] * n
    st: List[int] = []
    t = 0
    ncomp = 0
    for s in range(n):
        if order[s] != -1:
            continue
        frames = [(s, iter(adj[s]))]
        order[s] = low[s] = t
        t += 1
        st.append(s)
        onstack[s] = True
        while frames:
            v, it = frames[-1]
            pushed = False
            for w in it:
                if order[w] == -1:
                    order[w] = low[w] = t
                    t += 1
                    st.append(w)
                    onstack[w] = True
                    frames.append((w, iter(adj[w])))
                    pushed = True
                    break
                if onstack[w] and order[w] < low[v]:
                    low[v] = order[w]
            if pushed:
                continue
            frames.pop()
            if frames and low[v] < low[frames[-1][0]]:
                low[frames[-1][0]] = low[v]
            if low[v] == order[v]:
                while True:
                    w = st.pop()
                    onstack[w] = False
                    comp[w] = ncomp
                    if w == v:
                        break
                ncomp += 1
    return ncomp, comp


def scc_labeling(s: SparsePair, matching: Matching) -> SccLabeling:
    """Components of the digraph on matched pairs (preprocess.py:200-218):
    pair i = (row i, column row_to_col[i]); an unmatched entry (r, c) is the
    edge pair(col_to_row[c]) -> pair(r)."""
    n = s.n
    crs = s.crs
    adj: List[List[int]] = [[] for _ in range(n)]
    for r in range(n):
        for p in range(crs.rptrs[r], crs.rptrs[r + 1]):
            u = matching.col_to_row[crs.cids[p]]
            if u != r:
                adj[u].append(r)
    count, comp = strongly_connected(adj)
    return SccLabeling(count, tuple(comp), tuple(comp[matching.col_to_row[c]] for c in range(n)))


def dm_decompose(s: SparsePair) -> Union[DmResult, SingularVerdict]:
    """Matching filter of one sparse matrix (preprocess.py:221-240)."""
    m = max_matching(BipartiteGraph.from_sparse(s))
    if not m.perfect:
        return SingularVerdict(f"maximum matching has size {m.size} < {s.n}; permanent is 0")
    lab = scc_labeling(s, m)
    kept, removed = [], []
    for (r, c, v) in s.crs.triplets():
        if m.row_to_col[r] != c and lab.row_component[r] != lab.col_component[c]:
            removed.append((r, c))
        else:
            kept.append((r, c, v))
    nnz = s.crs.nnz
    if not removed:
        return DmResult(m, lab, (), s, nnz, nnz)
    return DmResult(m, lab, tuple(removed), sparse_from_triplets(s.n, kept, s.kind), nnz,
                    len(kept))


def dm_filter(s: SparsePair) -> Union[SparsePair, SingularVerdict]:
    """Permanent-preserving entry deletion; SingularVerdict when perm = 0."""
    res = dm_decompose(s)
    return res if isinstance(res, SingularVerdict) else res.filtered


# ---------------------------------------------------------------------------
# compressions on the row-list form


def _rows_of(s: SparsePair) -> Rows:
    crs = s.crs
    return [[(crs.cids[p], crs.vals[p]) for p in range(crs.rptrs[i], crs.rptrs[i + 1])]
            for i in range(s.n)]


def _pair_of(n: int, rows: Rows, kind: str) -> SparsePair:
    return sparse_from_triplets(n, [(i, j, v) for i, r in enumerate(rows) for (j, v) in r], kind)


def _col_counts(n: int, rows: Rows) -> List[int]:
    cnt = [0] * n
    for r in rows:
        for (j, _) in r:
            cnt[j] += 1
    return cnt


class MinNnz(NamedTuple):
    axis: str  # "row" or "col"
    index: int
    count: int


def _min_nnz(n: int, rows: Rows) -> MinNnz:
    best = MinNnz("row", 0, n + 1)
    for i, r in enumerate(rows):
        if len(r) < best.count:
            best = MinNnz("row", i, len(r))
    for j, c in enumerate(_col_counts(n, rows)):
        if c < best.count:
            best = MinNnz("col", j, c)
    return best


def min_nnz_row_col(s: SparsePair) -> MinNnz:
    """Sparsest row or column; rows win ties, then the lowest index
    (preprocess.py:257-270)."""
    return _min_nnz(s.n, _rows_of(s))


def _col_entries(rows: Rows, c: int) -> List[Tuple[int, Scalar]]:
    out = []
    for i, r in enumerate(rows):
        for (j, v) in r:
            if j == c:
                out.append((i, v))
                break
            if j > c:
                break
    return out


def _drop(rows: Rows, r: int, c: int) -> Rows:
    """Minor without row r and column c (indices above shift down)."""
    return [[(j - (j > c), v) for (j, v) in row if j != c] for i, row in enumerate(rows) if i != r]


def _fold_cols(rows: Rows, row: int, j1: int, a1, j2: int, a2) -> Rows:
    """Drop `row`; columns j1 < j2 become the single column a2*col(j1) +
    a1*col(j2) at index 0, the other columns keep their order after it
    (preprocess.py:304-326; same scalar operations in the same order)."""
    out = []
    for i, r in enumerate(rows):
        if i == row:
            continue
        comb = None
        rest = []
        for (j, v) in r:
            if j == j1:
                comb = (0 if comb is None else comb) + a2 * v
            elif j == j2:
                comb = (0 if comb is None else comb) + a1 * v
            else:
                rest.append((j + 1 - (j > j1) - (j > j2), v))
        if comb is not None and comb != 0:
            rest.insert(0, (0, comb))
        out.append(rest)
    return out


def _fold_rows(rows: Rows, col: int, i1: int, a1, i2: int, a2) -> Rows:
    """Transposed _fold_cols: drop column `col`; rows i1 < i2 become the
    single row a2*row(i1) + a1*row(i2) at index 0, the others follow in order."""
    comb: Dict[int, Scalar] = {}
    # the reference folds on the transpose, visiting each transposed row
    # (= original column) in ascending original-row order: i1 before i2
    for (j, v) in rows[i1]:
        if j != col:
            jj = j - (j > col)
            comb[jj] = comb.get(jj, 0) + a2 * v
    for (j, v) in rows[i2]:
        if j != col:
            jj = j - (j > col)
            comb[jj] = comb.get(jj, 0) + a1 * v
    first = [(j, v) for (j, v) in sorted(comb.items()) if v != 0]
    out = [first]
    for i, r in enumerate(rows):
        if i == i1 or i == i2:
            continue
        out.append([(j - (j > col), v) for (j, v) in r if j != col])
    return out


def _d1(rows: Rows, axis: str, index: int):
    if axis == "row":
        if len(rows[index]) != 1:
            raise StructureError(f"row {index} has {len(rows[index])} nonzeros, d1 needs 1")
        col, alpha = rows[index][0]
        return alpha, _drop(rows, index, col)
    ent = _col_entries(rows, index)
    if len(ent) != 1:
        raise StructureError(f"row {index} has {len(ent)} nonzeros, d1 needs 1")
    r, alpha = ent[0]
    return alpha, _drop(rows, r, index)


def _d2(rows: Rows, axis: str, index: int) -> Rows:
    if axis == "row":
        if len(rows[index]) != 2:
            raise StructureError(f"row {index} has {len(rows[index])} nonzeros, d2 needs 2")
        (j1, a1), (j2, a2) = rows[index]
        return _fold_cols(rows, index, j1, a1, j2, a2)
    ent = _col_entries(rows, index)
    if len(ent) != 2:
        raise StructureError(f"row {index} has {len(ent)} nonzeros, d2 needs 2")
    (i1, a1), (i2, a2) = ent
    return _fold_rows(rows, index, i1, a1, i2, a2)


def _d34(rows: Rows, axis: str, index: int) -> Tuple[Rows, Rows]:
    if axis == "row":
        ent = rows[index]
        if len(ent) < 3:
            raise StructureError(f"row {index} has {len(ent)} nonzeros, d34 needs >= 3")
        (j1, a1), (j2, a2) = ent[0], ent[1]
        zeroed = [r if i != index else r[2:] for i, r in enumerate(rows)]
        return zeroed, _fold_cols(rows, index, j1, a1, j2, a2)
    ent = _col_entries(rows, index)
    if len(ent) < 3:
        raise StructureError(f"row {index} has {len(ent)} nonzeros, d34 needs >= 3")
    (i1, a1), (i2, a2) = ent[0], ent[1]
    zeroed = [[(j, v) for (j, v) in r if j != index] if i in (i1, i2) else r
              for i, r in enumerate(rows)]
    return zeroed, _fold_rows(rows, index, i1, a1, i2, a2)


def d1compress(s: SparsePair, axis: str, index: int) -> Tuple[Scalar, SparsePair]:
    """Row/column with one nonzero: perm(A) = alpha * perm(minor), n >= 2
    (preprocess.py:289-301)."""
    if s.n < 2:
        raise StructureError("d1compress needs n >= 2")
    alpha, minor = _d1(_rows_of(s), axis, index)
    return alpha, _pair_of(s.n - 1, minor, s.kind)


def d2compress(s: SparsePair, axis: str, index: int) -> SparsePair:
    """Row/column with two nonzeros folds into an (n-1)-sized matrix
    (preprocess.py:329-339)."""
    if s.n < 2:
        raise StructureError("d2compress needs n >= 2")
    return _pair_of(s.n - 1, _d2(_rows_of(s), axis, index), s.kind)


def d34compress(s: SparsePair, axis: str, index: int) -> Tuple[SparsePair, SparsePair]:
    """Split on the two lowest-index nonzeros of a 3+ entry row/column:
    (same-size matrix without them, folded (n-1)-sized matrix); the two
    permanents sum to perm(A) (preprocess.py:342-364)."""
    if s.n < 2:
        raise StructureError("d34compress needs n >= 2")
    z, f = _d34(_rows_of(s), axis, index)
    return _pair_of(s.n, z, s.kind), _pair_of(s.n - 1, f, s.kind)


# ---------------------------------------------------------------------------
# decomposition driver


@dataclass(frozen=True)
class DecompTask:
    matrix: SparsePair
    multiplier: Scalar
    depth: int
    task_id: int


@dataclass
class DecompStats:
    tasks_created: int = 0
    d1_applied: int = 0
    d2_applied: int = 0
    d34_applied: int = 0
    trivial_leaves: int = 0
    kernel_leaves: int = 0
    dense_kernel_leaves: int = 0
    max_depth: int = 0
    elapsed: float = 0.0
    leaf_sizes: List[int] = field(default_factory=list)
    leaf_nnzs: List[int] = field(default_factory=list)
    leaf_launches: int = 0  # device calls issued for the kernel leaves

    @property
    def avg_leaf_n(self) -> float:
        return sum(self.leaf_sizes) / len(self.leaf_sizes) if self.leaf_sizes else 0.0

    @property
    def avg_leaf_nnz(self) -> float:
        return sum(self.leaf_nnzs) / len(self.leaf_nnzs) if self.leaf_nnzs else 0.0


def _combine_contributions(contribs: List[Tuple[int, Scalar]], kind: str) -> Scalar:
    """Leaf contributions in ascending task-id order, double-double
    (preprocess.py:398-417)."""
    contribs.sort(key=lambda t: t[0])
    if kind == KIND_INT:
        return sum(v for _, v in contribs)
    import numpy as np
    if kind == KIND_COMPLEX:
        vals = np.array([complex(v) for _, v in contribs], dtype=np.complex128)
        return complex(_dd_sum(np.ascontiguousarray(vals.real)),
                       _dd_sum(np.ascontiguousarray(vals.imag)))
    return _dd_sum(np.array([float(v) for _, v in contribs], dtype=np.float64))


def _dd_sum(vals) -> float:
    """hi of the in-order double-double sum of vals (one C call; the same
    dd_add sequence as the reference's loop)."""
    from . import _native as nat
    import numpy as np
    vals = np.ascontiguousarray(vals, dtype=np.float64)
    out = np.zeros(2)
    nat.check(nat.load().pk_dd_accumulate(nat.dptr(vals) if len(vals) else None, len(vals),
                                          nat.dptr(out)), "pk_dd_accumulate")
    return float(out[0])


class _LeafQueue:
    """Kernel leaves waiting for a batched device evaluation."""

    def __init__(self, kind: str, policy: AccumulatorPolicy, device: int, stats: DecompStats):
        # kind/policy/device of the whole tree; leaves of every order queue here
        self.kind, self.policy, self.device, self.stats = kind, policy, device, stats
        self.items: List[Tuple[int, Scalar, SparsePair]] = []

    def add(self, task_id: int, mult: Scalar, m: SparsePair, out: List[Tuple[int, Scalar]]):
        self.items.append((task_id, mult, m))
        if len(self.items) >= LEAF_BATCH:
            self.flush(out)

    def flush(self, out: List[Tuple[int, Scalar]]) -> None:
        if not self.items:
            return
        from .batch import permanent_batch
        from .integer import int_walk_total
        from .matrix import sparse_to_dense
        items, self.items = self.items, []
        if self.kind == KIND_INT:
            from .integer import int_batch_totals
            by_n: Dict[int, List[int]] = defaultdict(list)
            for k, (_, _, m) in enumerate(items):
                by_n[m.n].append(k)
            for n, idx in by_n.items():
                vals = int_batch_totals([sparse_to_dense(items[k][2]) for k in idx], self.device)
                self.stats.leaf_launches += 1
                for k, v in zip(idx, vals):
                    tid, mult, _ = items[k]
                    out.append((tid, mult * v))
            return
        groups: Dict[int, List[int]] = defaultdict(list)
        for k, (_, _, m) in enumerate(items):
            groups[m.n].append(k)
        for n, idx in groups.items():
            vals = permanent_batch([sparse_to_dense(items[k][2]) for k in idx], self.policy,
                                   device=self.device)
            self.stats.leaf_launches += 1
            for k, v in zip(idx, vals):
                tid, mult, _ = items[k]
                out.append((tid, mult * v))


def _decompose(s: SparsePair, stats: DecompStats, contribs: List[Tuple[int, Scalar]],
               on_leaf, task_limit: int, time_limit: float, min_nnz_threshold: int,
               dense_leaf_density: float) -> None:
    """The worklist of decomp_run (preprocess.py:442-504); kernel leaves go to
    on_leaf(task_id, multiplier, SparsePair)."""
    kind = s.kind
    one: Scalar = 1 if kind == KIND_INT else (complex(1.0) if kind == KIND_COMPLEX else 1.0)
    started = time.monotonic()
    # task = (n, rows, multiplier, depth, task id)
    stack = [(s.n, _rows_of(s), one, 0, 0)]
    next_id = 1
    stats.tasks_created = 1
    while stack:
        if stats.tasks_created > task_limit:
            raise DecompTimeout(f"task budget of {task_limit} exhausted",
                                tasks_done=stats.tasks_created,
                                elapsed=time.monotonic() - started)
        if time.monotonic() - started > time_limit:
            raise DecompTimeout(f"wall-clock budget of {time_limit:.1f}s exhausted",
                                tasks_done=stats.tasks_created,
                                elapsed=time.monotonic() - started)
        n, rows, mult, depth, tid = stack.pop()
        if depth > stats.max_depth:
            stats.max_depth = depth
        pick = _min_nnz(n, rows)
        if pick.count == 0:
            stats.trivial_leaves += 1  # empty row or column: contributes 0
            continue
        if n == 1:
            stats.trivial_leaves += 1
            contribs.append((tid, mult * rows[0][0][1]))
            continue
        if pick.count == 1:
            alpha, minor = _d1(rows, pick.axis, pick.index)
            stats.d1_applied += 1
            stack.append((n - 1, minor, mult * alpha, depth + 1, next_id))
            next_id += 1
            stats.tasks_created += 1
            continue
        if pick.count == 2:
            stats.d2_applied += 1
            stack.append((n - 1, _d2(rows, pick.axis, pick.index), mult, depth + 1, next_id))
            next_id += 1
            stats.tasks_created += 1
            continue
        if pick.count <= min_nnz_threshold:
            zeroed, folded = _d34(rows, pick.axis, pick.index)
            stats.d34_applied += 1
            stack.append((n, zeroed, mult, depth + 1, next_id))
            stack.append((n - 1, folded, mult, depth + 1, next_id + 1))
            next_id += 2
            stats.tasks_created += 2
            continue
        # dense enough everywhere: a kernel leaf
        nnz = sum(len(r) for r in rows)
        stats.kernel_leaves += 1
        stats.leaf_sizes.append(n)
        stats.leaf_nnzs.append(nnz)
        if nnz / (n * n) >= dense_leaf_density:
            stats.dense_kernel_leaves += 1
        on_leaf(tid, mult, _pair_of(n, rows, kind))
    stats.elapsed = time.monotonic() - started


def _native_tree(s: SparsePair, task_limit: int, time_limit: float, min_nnz_threshold: int,
                 dense_leaf_density: float):
    """The task tree from the native worklist (csrc/pk_decomp.cu): (trivial
    contributions, leaves grouped by order {n: (task ids, multipliers,
    matrices[b, n, n])}, stats); None when the integers outgrow 128 bits
    (the Python worklist then takes over with arbitrary precision)."""
    import ctypes

    import numpy as np

    from . import _native as nat
    from .matrix import sparse_to_dense
    n, kind = s.n, s.kind
    dense = sparse_to_dense(s)
    if kind == KIND_INT:
        code, dt, width = nat.PK_KIND_INT, np.int64, 2
        a = np.array([int(v) for v in dense.data], dtype=object)
        if any(abs(int(v)) >= (1 << 63) for v in a):
            return None
        a = np.ascontiguousarray(a.astype(np.int64))
    elif kind == KIND_COMPLEX:
        code, dt, width = nat.PK_KIND_COMPLEX, np.float64, 2
        a = np.ascontiguousarray(np.array(dense.data, dtype=np.complex128).view(np.float64))
    else:
        code, dt, width = nat.PK_KIND_REAL, np.float64, 1
        a = np.ascontiguousarray(np.array(dense.data, dtype=np.float64))
    lib = nat.load()
    h = ctypes.c_void_p()
    res = nat.DecompResult()
    rc = lib.pk_decomp_tree(code, n, a.ctypes.data_as(ctypes.c_void_p), min_nnz_threshold,
                            task_limit, time_limit, dense_leaf_density, ctypes.byref(h),
                            ctypes.byref(res))
    if rc == nat.PK_ERR_OVERFLOW:
        return None
    if rc == nat.PK_ERR_TIMEOUT:
        raise DecompTimeout(lib.pk_decomp_last_error().decode(),
                            tasks_done=int(res.stats.tasks_created))
    if rc != nat.PK_OK:
        raise StructureError(lib.pk_decomp_last_error().decode())
    try:
        nt, nl, nv = int(res.trivial), int(res.leaves), int(res.leaf_values)
        t_id = np.zeros(max(nt, 1), dtype=np.int64)
        t_val = np.zeros(max(nt, 1) * width, dtype=dt)
        l_id = np.zeros(max(nl, 1), dtype=np.int64)
        l_n = np.zeros(max(nl, 1), dtype=np.int32)
        l_mult = np.zeros(max(nl, 1) * width, dtype=dt)
        l_vals = np.zeros(max(nv, 1) * width, dtype=dt)
        vp = lambda x: x.ctypes.data_as(ctypes.c_void_p)
        lib.pk_decomp_fetch(h, nat.i64ptr(t_id), vp(t_val), nat.i64ptr(l_id), nat.i32ptr(l_n),
                            vp(l_mult), vp(l_vals))
    finally:
        lib.pk_decomp_free(h)

    def scalar(arr, k):
        if kind == KIND_INT:
            lo, hi = int(arr[2 * k]) & ((1 << 64) - 1), int(arr[2 * k + 1])
            return (hi << 64) | lo
        if kind == KIND_COMPLEX:
            return complex(float(arr[2 * k]), float(arr[2 * k + 1]))
        return float(arr[k])

    trivial = [(int(t_id[k]), scalar(t_val, k)) for k in range(nt)]
    groups: Dict[int, Tuple[List[int], List[Scalar], List[int]]] = defaultdict(
        lambda: ([], [], []))
    off = 0
    for k in range(nl):
        m = int(l_n[k])
        g = groups[m]
        g[0].append(int(l_id[k]))
        g[1].append(scalar(l_mult, k))
        g[2].append(off)
        off += m * m
    leaves = {}
    for m, (ids, mults, offs) in groups.items():
        if kind == KIND_INT:
            vals = l_vals.reshape(-1, 2)
            mats = [[[scalar(l_vals, o + i * m + j) for j in range(m)] for i in range(m)]
                    for o in offs]
        elif kind == KIND_COMPLEX:
            c = l_vals.view(np.complex128)
            mats = np.stack([c[o:o + m * m].reshape(m, m) for o in offs])
        else:
            mats = np.stack([l_vals[o:o + m * m].reshape(m, m) for o in offs])
        leaves[m] = (ids, mults, mats)
    st = res.stats
    stats = DecompStats(tasks_created=int(st.tasks_created), d1_applied=int(st.d1_applied),
                        d2_applied=int(st.d2_applied), d34_applied=int(st.d34_applied),
                        trivial_leaves=int(st.trivial_leaves), kernel_leaves=int(st.kernel_leaves),
                        dense_kernel_leaves=int(st.dense_kernel_leaves),
                        max_depth=int(st.max_depth))
    for m, (ids, _, _) in leaves.items():
        stats.leaf_sizes.extend([m] * len(ids))
    return trivial, leaves, stats


def _evaluate_native_leaves(leaves, kind, policy, device, stats, contribs) -> None:
    """Batched device evaluation of the native tree's leaves (one launch per
    order for real / complex; exact integer kernels per leaf)."""
    from .batch import complex_batch_arrays, real_batch_arrays
    from .integer import int_walk_total
    from .matrix import DenseMatrix
    for m, (ids, mults, mats) in sorted(leaves.items()):
        if kind == KIND_INT:
            from .integer import int_batch_totals
            for lo in range(0, len(ids), LEAF_BATCH):
                vals = int_batch_totals([DenseMatrix.from_rows(r, kind=KIND_INT)
                                         for r in mats[lo:lo + LEAF_BATCH]], device)
                stats.leaf_launches += 1
                for tid, mult, v in zip(ids[lo:lo + LEAF_BATCH], mults[lo:lo + LEAF_BATCH], vals):
                    contribs.append((tid, mult * v))
            continue
        for lo in range(0, len(ids), LEAF_BATCH):
            chunk = mats[lo:lo + LEAF_BATCH]
            if kind == KIND_COMPLEX and m <= 40:
                if policy is not AccumulatorPolicy.DD:
                    from .errors import PolicyError
                    raise PolicyError("complex matrices support the plain-double policy only")
                vals = complex_batch_arrays(chunk, device)
            elif kind == KIND_COMPLEX:
                from .batch import permanent_batch
                vals = permanent_batch([DenseMatrix.from_array(x) for x in chunk], policy,
                                       device=device)
            else:
                vals = real_batch_arrays(chunk, policy, device)
            stats.leaf_launches += 1
            for tid, mult, v in zip(ids[lo:lo + LEAF_BATCH], mults[lo:lo + LEAF_BATCH], vals):
                contribs.append((tid, mult * v))


def decomp_run(s: SparsePair, policy: "AccumulatorPolicy | str" = AccumulatorPolicy.DD,
               task_limit: int = DEFAULT_TASK_LIMIT, time_limit: float = DEFAULT_TIME_LIMIT,
               min_nnz_threshold: int = 4, dense_leaf_density: float = DENSE_LEAF_DENSITY,
               *, device: int = 0, native: bool = True) -> Tuple[Scalar, DecompStats]:
    """Worklist compression driver; returns (permanent, statistics)
    (preprocess.py:420-507). Tasks are processed LIFO; exceeding the task or
    wall-clock budget raises DecompTimeout with progress attached.

    The task tree is walked by the native worklist (csrc/pk_decomp.cu; the
    Python one below when native=False or integers outgrow 128 bits), and
    kernel leaves are evaluated in batched launches on `device` (module
    docstring); every leaf goes to the dense batched kernels (x + 0 == x: the
    sparse walk's arithmetic), its density only feeds the statistics."""
    policy = as_policy(policy)
    started = time.monotonic()
    contribs: List[Tuple[int, Scalar]] = []
    tree = _native_tree(s, task_limit, time_limit, min_nnz_threshold,
                        dense_leaf_density) if native else None
    if tree is not None:
        trivial, leaves, stats = tree
        contribs.extend(trivial)
        _evaluate_native_leaves(leaves, s.kind, policy, device, stats, contribs)
    else:
        stats = DecompStats()
        leaves_q = _LeafQueue(s.kind, policy, device, stats)
        _decompose(s, stats, contribs, lambda t, m, a: leaves_q.add(t, m, a, contribs),
                   task_limit, time_limit, min_nnz_threshold, dense_leaf_density)
        leaves_q.flush(contribs)
    stats.elapsed = time.monotonic() - started
    return _combine_contributions(contribs, s.kind), stats


def decomp_ryser(s: SparsePair, policy: "AccumulatorPolicy | str" = AccumulatorPolicy.DD,
                 task_limit: int = DEFAULT_TASK_LIMIT,
                 time_limit: float = DEFAULT_TIME_LIMIT) -> Scalar:
    """Compression-first permanent of a sparse matrix (preprocess.py:510-518)."""
    value, _ = decomp_run(s, policy, task_limit, time_limit)
    return value


def decomp_leaves(s: SparsePair, min_nnz_threshold: int = 4,
                  task_limit: int = DEFAULT_TASK_LIMIT,
                  dense_leaf_density: float = DENSE_LEAF_DENSITY):
    """The host half of decomp_run, no device work: (kernel leaves as
    (task id, multiplier, SparsePair) in permkit's evaluation order, trivial
    contributions, statistics). The CPU tests compare this task tree with
    the reference's own leaves."""
    stats = DecompStats()
    contribs: List[Tuple[int, Scalar]] = []
    out: List[Tuple[int, Scalar, SparsePair]] = []
    _decompose(s, stats, contribs, lambda t, m, a: out.append((t, m, a)), task_limit,
               float("inf"), min_nnz_threshold, dense_leaf_density)
    return out, contribs, stats
