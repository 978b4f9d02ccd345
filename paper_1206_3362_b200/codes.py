"""Parity-check matrices on the host: storage, structure detection, constructors.

This is the host side of the code handle.  `ParityCheckMatrix` mirrors the
reference's storage contract (`/root/reference/pkg/src/fwbf/matrix.py:22-58`):
``row_adj[m]`` is the sorted column list of check m, ``col_adj[n]`` the sorted
check list of bit n (ascending, because it is built row by row), plus the
row-major edge list.  Nothing here runs per frame; the decoder only sees the
device descriptor built from it (see `paper_1206_3362_b200.decoders`).

Constructors cover the five configurations of BASELINE.json:
  * `eg_ldpc(s)`       type-I cyclic EG(2, 2^s) codes, the reference's algorithm
                       (`eg.py:9-47`, `gf.py:88-92`) extended to s = 6;
  * `qc_ldpc(...)`     quasi-cyclic (j, k) array of circulant shifts with 4-cycles
                       rejected (not in the reference: SPEC.md:107 non-goal);
  * `gallager_rc(...)` a (dv, dc)-regular 4-cycle-free code by greedy placement.
"""

from __future__ import annotations

import os
from dataclasses import dataclass
from typing import Iterable, List, Optional, Sequence

import numpy as np

__all__ = [
    "ParityCheckMatrix", "CodeStructure", "detect_structure", "eg_ldpc",
    "qc_ldpc", "gallager_rc", "gf2_rank", "validate_rc", "code_dimension",
    "write_alist", "read_alist", "AlistError", "AlistFormatError", "AlistRangeError",
    "AlistMismatchError", "CodeSpec", "code_spec", "RcReport",
]


class ParityCheckMatrix:
    """M x N binary matrix kept as sorted row and column adjacency lists.

    Same contract as the reference (`matrix.py:22-58`): rows are sorted and
    duplicate-free; ``col_adj[n]`` lists checks in ascending order; ``edge_row``
    / ``edge_col`` enumerate the ones row-major.  Immutable after construction.
    """

    def __init__(self, row_adj: Sequence[Iterable[int]], n_cols: int):
        if n_cols < 1:
            raise ValueError("n_cols must be positive")
        rows: List[np.ndarray] = []
        for m, adj in enumerate(row_adj):
            raw = np.asarray(list(adj), dtype=np.int64).ravel()
            arr = np.unique(raw)
            if arr.size != raw.size:
                raise ValueError(f"row {m} has a duplicate column index")
            if arr.size and (arr[0] < 0 or arr[-1] >= n_cols):
                raise ValueError(f"row {m} has a column index out of range")
            rows.append(arr)
        self.n_rows = len(rows)
        self.n_cols = int(n_cols)
        self.row_adj = tuple(rows)
        self.row_weights = np.array([r.size for r in rows], dtype=np.int64)
        self.edge_row = np.repeat(np.arange(self.n_rows, dtype=np.int64), self.row_weights)
        self.edge_col = np.concatenate(rows) if rows else np.zeros(0, np.int64)
        # Column view: a stable sort by column keeps checks ascending per column.
        order = np.argsort(self.edge_col, kind="stable")
        self.col_weights = np.bincount(self.edge_col, minlength=self.n_cols).astype(np.int64)
        col_ptr = np.zeros(self.n_cols + 1, np.int64)
        np.cumsum(self.col_weights, out=col_ptr[1:])
        self.col_ptr = col_ptr
        self.col_idx = self.edge_row[order]
        self.col_adj = tuple(self.col_idx[col_ptr[n]:col_ptr[n + 1]] for n in range(self.n_cols))
        row_ptr = np.zeros(self.n_rows + 1, np.int64)
        np.cumsum(self.row_weights, out=row_ptr[1:])
        self.row_ptr = row_ptr
        self.max_row_weight = int(self.row_weights.max()) if self.n_rows else 0
        self.max_col_weight = int(self.col_weights.max()) if self.n_cols else 0

    @classmethod
    def from_dense(cls, a) -> "ParityCheckMatrix":
        a = np.asarray(a)
        return cls([np.nonzero(a[m])[0] for m in range(a.shape[0])], a.shape[1])

    def to_dense(self) -> np.ndarray:
        out = np.zeros((self.n_rows, self.n_cols), dtype=np.uint8)
        out[self.edge_row, self.edge_col] = 1
        return out

    @property
    def n_edges(self) -> int:
        return int(self.edge_col.size)

    @property
    def row_pad(self) -> np.ndarray:
        """[M, max row weight] column indices padded with the sentinel N (matrix.py:53-58)."""
        pad = np.full((self.n_rows, self.max_row_weight), self.n_cols, dtype=np.int64)
        for m, arr in enumerate(self.row_adj):
            pad[m, :arr.size] = arr
        return pad

    def transpose(self) -> "ParityCheckMatrix":
        return ParityCheckMatrix(self.col_adj, self.n_rows)

    def syndrome(self, z) -> np.ndarray:
        """z H^T over GF(2) (reference `matrix.py:72-79`)."""
        z = np.asarray(z)
        if z.shape != (self.n_cols,):
            raise ValueError(f"expected a length-{self.n_cols} vector")
        par = np.bitwise_xor.reduceat(z[self.edge_col].astype(np.uint8), self.row_ptr[:-1]) \
            if self.n_edges else np.zeros(self.n_rows, np.uint8)
        par = np.where(self.row_weights > 0, par, 0)
        return par.astype(np.uint8)

    def __eq__(self, other) -> bool:
        if not isinstance(other, ParityCheckMatrix):
            return NotImplemented
        return (self.n_rows == other.n_rows and self.n_cols == other.n_cols
                and all(np.array_equal(a, b) for a, b in zip(self.row_adj, other.row_adj)))

    def __repr__(self) -> str:
        return f"ParityCheckMatrix({self.n_rows}x{self.n_cols}, {self.n_edges} ones)"


# --------------------------------------------------------------------------
# Structure detection: the device descriptor is cheapest for circulant and
# quasi-cyclic matrices (index arithmetic instead of index tables).
# --------------------------------------------------------------------------

@dataclass(frozen=True)
class CodeStructure:
    kind: str                        # "circulant" | "qc" | "explicit"
    offsets: Optional[np.ndarray] = None   # circulant: sorted first-row columns
    z: int = 0                       # qc: circulant size
    shifts: Optional[np.ndarray] = None    # qc: [jb, kb] shifts, -1 = zero block


def detect_structure(h: ParityCheckMatrix) -> CodeStructure:
    """Classify H.  Circulant: square, row m = row 0 shifted by m (eg.py:46).
    QC: every Z x Z block is zero or one shifted identity (row i -> col i+s)."""
    n, m = h.n_cols, h.n_rows
    if n == m and h.n_rows > 0:
        first = h.row_adj[0]
        w = first.size
        if w and np.all(h.row_weights == w):
            rows = np.sort((first[None, :] + np.arange(m)[:, None]) % n, axis=1)
            if np.array_equal(rows.ravel(), h.edge_col):
                return CodeStructure("circulant", offsets=first.astype(np.int64))
    for z in _qc_candidates(h):
        st = _try_qc(h, z)
        if st is not None:
            return st
    return CodeStructure("explicit")


def _qc_candidates(h: ParityCheckMatrix):
    g = np.gcd(h.n_rows, h.n_cols)
    cands = [d for d in (1024, 512, 256, 128, 64, 32, 16) if g % d == 0 and d < h.n_cols]
    return cands


def _try_qc(h: ParityCheckMatrix, z: int) -> Optional[CodeStructure]:
    jb, kb = h.n_rows // z, h.n_cols // z
    shifts = np.full((jb, kb), -1, np.int64)
    rows = h.edge_row
    cols = h.edge_col
    br, bc = rows // z, cols // z
    s = (cols % z - rows % z) % z
    key = br * kb + bc
    # each block must hold exactly z ones, all with the same shift
    cnt = np.bincount(key, minlength=jb * kb)
    if np.any((cnt != 0) & (cnt != z)):
        return None
    first = np.full(jb * kb, -1, np.int64)
    first[key[::-1]] = s[::-1]
    if np.any(first[key] != s):
        return None
    shifts.ravel()[:] = np.where(cnt == z, first, -1)
    return CodeStructure("qc", z=z, shifts=shifts)


# --------------------------------------------------------------------------
# GF(2^m) and EG-LDPC construction (reference gf.py:29-92, eg.py:9-47).
# --------------------------------------------------------------------------

# Lin & Costello primitive polynomials, bit i = coefficient of x^i
# (same published table as gf.py:10-26).
_PRIM_POLY = {2: 0x7, 3: 0xB, 4: 0x13, 5: 0x25, 6: 0x43, 7: 0x89, 8: 0x11D,
              9: 0x211, 10: 0x409, 11: 0x805, 12: 0x1053, 13: 0x201B,
              14: 0x4443, 15: 0x8003, 16: 0x1100B}


def _gf_tables(m: int):
    order = 1 << m
    poly = _PRIM_POLY[m]
    exp = np.zeros(order - 1, np.int64)
    log = np.full(order, -1, np.int64)
    x = 1
    for i in range(order - 1):
        exp[i] = x
        log[x] = i
        x <<= 1
        if x & order:
            x ^= poly
    if x != 1 or np.any(log[1:] < 0):
        raise ValueError(f"polynomial for m={m} is not primitive")
    return exp, log


def eg_ldpc(s: int) -> ParityCheckMatrix:
    """Type-I cyclic EG(2, 2^s) LDPC matrix, n = 4^s - 1, weight 2^s.

    Same deterministic choices as the reference (`eg.py:22-47`): points are
    powers of alpha in GF(2^(2s)); the base line is {a + beta*b : beta in GF(2^s)}
    with (log a, log b) the first pair in scan order whose log difference is not
    a multiple of 2^s + 1; rows are the n cyclic shifts of that line.  The
    reference guards s <= 5 (`eg.py:20-21`); s = 6 gives the (4095, 3367) code.
    """
    if s not in (2, 3, 4, 5, 6):
        raise ValueError(f"geometry parameter s must be in 2..6, got {s}")
    m = 2 * s
    exp, log = _gf_tables(m)
    n = (1 << m) - 1
    q = 1 << s
    stride = q + 1
    sub = [0] + [int(exp[(stride * t) % n]) for t in range(q - 1)]
    # First (i, j) in row-major scan with (i - j) mod n not a multiple of stride:
    # i = 0 and j = 1 always qualifies because stride > 1.
    base_i, base_j = 0, 1
    a, b = int(exp[base_i]), int(exp[base_j])

    def gmul(u, v):
        if u == 0 or v == 0:
            return 0
        return int(exp[(log[u] + log[v]) % n])

    line = [a ^ gmul(beta, b) for beta in sub]
    if len(set(line)) != q or 0 in line:
        raise AssertionError("base line construction failed")
    first = np.sort(np.array([log[x] for x in line], np.int64))
    rows = [(first + i) % n for i in range(n)]
    return ParityCheckMatrix(rows, n)


# --------------------------------------------------------------------------
# Quasi-cyclic (j, k) codes and RC-free regular Gallager codes (builder-made;
# the reference cannot construct them).
# --------------------------------------------------------------------------

def qc_shifts(jb: int, kb: int, z: int, seed: int) -> np.ndarray:
    """Seeded jb x kb circulant shift table with no 4-cycles.

    A 4-cycle through block rows r1, r2 and block columns c1, c2 exists iff
    s[r1,c1] - s[r2,c1] == s[r1,c2] - s[r2,c2] (mod z).  Columns are drawn one
    at a time; a draw is kept only if, for every row pair, its difference is new.
    """
    rng = np.random.default_rng(seed)
    shifts = np.zeros((jb, kb), np.int64)
    used = [[set() for _ in range(jb)] for _ in range(jb)]
    for c in range(kb):
        for _attempt in range(10000):
            col = rng.integers(0, z, size=jb)
            ok = True
            for r1 in range(jb):
                for r2 in range(r1 + 1, jb):
                    if (col[r1] - col[r2]) % z in used[r1][r2]:
                        ok = False
                        break
                if not ok:
                    break
            if ok:
                break
        else:
            raise RuntimeError("could not place a 4-cycle-free column")
        for r1 in range(jb):
            for r2 in range(r1 + 1, jb):
                used[r1][r2].add(int((col[r1] - col[r2]) % z))
        shifts[:, c] = col
    return shifts


def qc_from_shifts(shifts: np.ndarray, z: int) -> ParityCheckMatrix:
    """Row r*z + i holds column c*z + (i + s[r, c]) mod z for every block."""
    jb, kb = shifts.shape
    rows = []
    i = np.arange(z)
    for r in range(jb):
        cols = np.stack([c * z + (i + shifts[r, c]) % z for c in range(kb) if shifts[r, c] >= 0], 1)
        rows.extend(np.sort(cols, axis=1))
    return ParityCheckMatrix(rows, kb * z)


def qc_ldpc(jb: int = 4, kb: int = 32, z: int = 512, seed: int = 2012) -> ParityCheckMatrix:
    """(jb, kb)-regular quasi-cyclic code of length kb*z, 4-cycle free."""
    return qc_from_shifts(qc_shifts(jb, kb, z, seed), z)


def gallager_rc(n: int = 504, dv: int = 3, dc: int = 6, seed: int = 1) -> ParityCheckMatrix:
    """(dv, dc)-regular code with no two columns sharing two checks.

    Columns are placed one at a time; each picks dv checks among those with
    spare degree, preferring the least-filled, and never a check that already
    shares a bit with another check picked for this column.  Restarts with a
    derived seed if it paints itself into a corner.
    """
    if (n * dv) % dc:
        raise ValueError("n*dv must be divisible by dc")
    m = n * dv // dc
    for attempt in range(200):
        rng = np.random.default_rng([seed, attempt])
        deg = np.zeros(m, np.int64)
        share = np.zeros((m, m), bool)     # share[a, b]: checks a, b meet in a bit
        cols: List[List[int]] = []
        ok = True
        for _c in range(n):
            chosen: List[int] = []
            for _k in range(dv):
                cand = np.nonzero(deg < dc)[0]
                if chosen:
                    bad = share[chosen].any(axis=0) | np.isin(np.arange(m), chosen)
                    cand = cand[~bad[cand]]
                if cand.size == 0:
                    ok = False
                    break
                low = cand[deg[cand] == deg[cand].min()]
                pick = int(rng.choice(low))
                chosen.append(pick)
            if not ok:
                break
            for a in chosen:
                deg[a] += 1
                for b in chosen:
                    if a != b:
                        share[a, b] = True
            cols.append(chosen)
        if ok and np.all(deg == dc):
            rows: List[List[int]] = [[] for _ in range(m)]
            for c, chk in enumerate(cols):
                for a in chk:
                    rows[a].append(c)
            return ParityCheckMatrix(rows, n)
    raise RuntimeError("greedy RC-free construction failed")


# --------------------------------------------------------------------------
# GF(2) rank, RC check, alist I/O (reference matrix.py:108-173, alist.py).
# --------------------------------------------------------------------------

def gf2_rank(h: ParityCheckMatrix) -> int:
    """Rank over GF(2) by Gaussian elimination on bit-packed uint64 rows."""
    if h.n_rows == 0:
        return 0
    words = (h.n_cols + 63) // 64
    a = np.zeros((h.n_rows, words), np.uint64)
    np.bitwise_or.at(a, (h.edge_row, h.edge_col // 64),
                     np.left_shift(np.uint64(1), (h.edge_col % 64).astype(np.uint64)))
    rank = 0
    rows_left = a
    for col in range(h.n_cols):
        if rows_left.shape[0] == 0:
            break
        w, b = divmod(col, 64)
        bit = np.uint64(1) << np.uint64(b)
        has = (rows_left[:, w] & bit) != 0
        idx = np.nonzero(has)[0]
        if idx.size == 0:
            continue
        piv = rows_left[idx[0]].copy()
        others = idx[1:]
        rows_left[others] ^= piv
        rows_left = np.delete(rows_left, idx[0], axis=0)
        rank += 1
    return rank


def code_dimension(h: ParityCheckMatrix) -> int:
    return h.n_cols - gf2_rank(h)


@dataclass(frozen=True)
class CodeSpec:
    """Block length, dimension, rate and (regular) weights of H (matrix.py:96-105)."""

    n: int
    k: int
    rate: float
    row_weight: Optional[int]  # None: irregular
    col_weight: Optional[int]


def code_spec(h: ParityCheckMatrix) -> CodeSpec:
    """(n, k = n - rank_GF2(H), k/n, weights) -- matrix.py:127-134; a degenerate
    code (k = 0 or k = n) raises ValueError."""
    k = code_dimension(h)
    if k <= 0 or k >= h.n_cols:
        raise ValueError(f"degenerate code: n={h.n_cols}, k={k}")
    rws, cws = np.unique(h.row_weights), np.unique(h.col_weights)
    return CodeSpec(n=h.n_cols, k=k, rate=k / h.n_cols,
                    row_weight=int(rws[0]) if rws.size == 1 else None,
                    col_weight=int(cws[0]) if cws.size == 1 else None)


@dataclass(frozen=True)
class RcReport:
    """Row-column constraint check (matrix.py:137-143): ``ok`` plus the
    lexicographically smallest pair of rows and of columns that share two or
    more positions.  Truthy iff ok."""

    ok: bool
    row_pair: Optional[tuple]
    col_pair: Optional[tuple]

    def __bool__(self) -> bool:
        return bool(self.ok)


def _smallest_shared_pair(lists: Sequence[np.ndarray], universe: int) -> Optional[tuple]:
    """Smallest (a, b), a < b, of items co-occurring in two or more of `lists`
    (each sorted): every list contributes its item pairs a * universe + b; a
    duplicated key is a pair seen twice."""
    keys = []
    for lst in lists:
        lst = np.asarray(lst, dtype=np.int64)
        if lst.size > 1:
            a, b = np.triu_indices(lst.size, 1)
            keys.append(lst[a] * universe + lst[b])
    if not keys:
        return None
    k = np.sort(np.concatenate(keys))
    dup = k[1:][k[1:] == k[:-1]]
    if dup.size == 0:
        return None
    first = int(dup[0])
    return (first // universe, first % universe)


def validate_rc(h: ParityCheckMatrix) -> RcReport:
    """No two rows, and no two columns, share more than one position."""
    rows = _smallest_shared_pair(h.col_adj, h.n_rows)   # rows co-occurring in two columns
    cols = _smallest_shared_pair(h.row_adj, h.n_cols)   # columns co-occurring in two rows
    return RcReport(ok=rows is None and cols is None, row_pair=rows, col_pair=cols)


class AlistError(ValueError):
    """An alist file could not be parsed (alist.py:19-20)."""


class AlistFormatError(AlistError):
    """Bad tokens, line counts or weights (alist.py:23-24)."""


class AlistRangeError(AlistError):
    """An index outside [1, M] or [1, N] (alist.py:27-28)."""


class AlistMismatchError(AlistError):
    """Column-side and row-side lists disagree (alist.py:31-32)."""


def write_alist(h: ParityCheckMatrix, path: str | os.PathLike) -> None:
    """Layout of `alist.py:35-44`: N M / maxima / weights / 1-based lists."""
    with open(path, "w", encoding="ascii", newline="\n") as f:
        f.write(f"{h.n_cols} {h.n_rows}\n{h.max_col_weight} {h.max_row_weight}\n")
        f.write(" ".join(map(str, h.col_weights.tolist())) + "\n")
        f.write(" ".join(map(str, h.row_weights.tolist())) + "\n")
        for adj in h.col_adj:
            f.write(" ".join(str(int(v) + 1) for v in adj) + "\n")
        for adj in h.row_adj:
            f.write(" ".join(str(int(v) + 1) for v in adj) + "\n")


def _alist_ints(line: str, lineno: int) -> List[int]:
    try:
        return [int(t) for t in line.split()]
    except ValueError:
        bad = next(t for t in line.split() if not t.lstrip("+-").isdigit())
        raise AlistFormatError(f"line {lineno}: non-integer token {bad!r}") from None


def _alist_lists(lines: Sequence[str], lineno0: int, weights: Sequence[int], wmax: int, bound: int,
                 what: str) -> List[List[int]]:
    """One 1-based index list per line, zero padding dropped; checked against the
    declared weights and range (alist.py:57-78)."""
    out = []
    for i, line in enumerate(lines):
        ln = lineno0 + i
        toks = _alist_ints(line, ln)
        if len(toks) > wmax:
            raise AlistFormatError(f"line {ln}: {what} {i} lists more than max weight {wmax} entries")
        vals = [v for v in toks if v]
        if len(vals) != weights[i]:
            raise AlistFormatError(f"line {ln}: {what} {i} declares weight {weights[i]} "
                                   f"but lists {len(vals)} indices")
        for v in vals:
            if v < 1 or v > bound:
                raise AlistRangeError(f"line {ln}: index {v} out of range [1, {bound}]")
        if len(set(vals)) != len(vals):
            raise AlistFormatError(f"line {ln}: {what} {i} has duplicate indices")
        out.append(sorted(v - 1 for v in vals))
    return out


def read_alist(path: str | os.PathLike) -> ParityCheckMatrix:
    """Parse an alist file (alist.py:81-128): header, weights, then the column
    and row lists; every failure is an AlistError subclass (a ValueError)."""
    with open(path, "r", encoding="ascii") as f:
        lines = f.read().split("\n")
    while lines and not lines[-1].strip():
        lines.pop()
    if len(lines) < 4:
        raise AlistFormatError("file has fewer than 4 header lines")
    head = _alist_ints(lines[0], 1)
    if len(head) != 2:
        raise AlistFormatError("line 1: expected 'N M'")
    n, m = head
    if n < 1 or m < 1:
        raise AlistFormatError(f"line 1: non-positive dimensions {n} x {m}")
    mx = _alist_ints(lines[1], 2)
    if len(mx) != 2:
        raise AlistFormatError("line 2: expected 'max_col_weight max_row_weight'")
    cw, rw = _alist_ints(lines[2], 3), _alist_ints(lines[3], 4)
    if len(cw) != n:
        raise AlistFormatError(f"line 3: expected {n} column weights, got {len(cw)}")
    if len(rw) != m:
        raise AlistFormatError(f"line 4: expected {m} row weights, got {len(rw)}")
    if min(cw) < 0 or max(cw) > mx[0]:
        raise AlistFormatError("line 3: a column weight exceeds the declared maximum")
    if min(rw) < 0 or max(rw) > mx[1]:
        raise AlistFormatError("line 4: a row weight exceeds the declared maximum")
    if len(lines) != 4 + n + m:
        raise AlistFormatError(f"expected {4 + n + m} lines, got {len(lines)}")
    col_lists = _alist_lists(lines[4:4 + n], 5, cw, mx[0], m, "column")
    row_lists = _alist_lists(lines[4 + n:], 5 + n, rw, mx[1], n, "row")
    seen = [[] for _ in range(m)]
    for col, rows in enumerate(col_lists):
        for r in rows:
            seen[r].append(col)
    for r in range(m):
        if seen[r] != row_lists[r]:  # both ascending
            raise AlistMismatchError(f"row {r}: column-side adjacency {seen[r]} "
                                     f"!= row-side adjacency {row_lists[r]}")
    return ParityCheckMatrix(row_lists, n)
