"""Seeded synthetic inputs shaped like the paper's workloads (BASELINE.json configs).

This module holds *input generation only* -- none of the method's arithmetic.
Both sides of every parity check (the CPU oracle in ``oracle/`` and the CUDA
path in ``paper_1606_04809_b200``) consume the arrays it returns; neither side
imports the other.

The paper's datasets (RCV1, URL, Covtype; Table 1, Table 2
P:1896-1910) are not available here, so these generators stand in for them
with the shapes, row-length spreads and column-popularity skew the paper
reports.  No record of those datasets is reproduced.  Recipe (DESIGN.md
"Input recipe"):

* RNG: ``SeedSequence(160604809 + k).spawn(3)`` -> (matrix, w*, label-noise)
  PCG64 streams, k = config number (1..4).
* every row is unit l2-normalised; labels y = sign(a.w* + 0.1 N(0,1)),
  w* ~ N(0, I_d), sign(0) := +1 (reading R10); lambda = 1/n.
* c1 tiny      n=1,000  d=100: each entry Bernoulli(0.1) (empty rows redrawn), N(0,1) values.
* c2 covtype   n=581,012 d=54: 10 continuous N(0,1) columns + one-hot(4) + one-hot(40)
                -> exactly 12 nnz/row (Table 2: 8/11.88/12).
* c3 rcv1      n=697,641 d=47,236: row length clip(round(LogNormal(ln 73.2 - s^2/2, s=0.63)),
                4, 1224); distinct columns = the first l distinct draws of an i.i.d.
                Zipf(1.1) stream over ranks 1..d; ranks are mapped to column ids by a
                seeded permutation (hot features are scattered, as in real data);
                values |N(0,1)| (tf-idf-like).
* c4 url       n=2,396,130 d=3,231,961: length clip(round(LogNormal(ln 115.6 - s^2/2,
                s=0.26)), 16, 414); Zipf(1.0) columns as above; values 1.0 w.p. 0.9
                else N(0,1).
``n_rows`` shrinks a config (same recipe, same d) for oracle-sized parity tests.
"""
from __future__ import annotations

import dataclasses
import hashlib
import os

import numpy as np

BASE_SEED = 160604809
SAMPLE_SEED = 160604809  # Philox key of the sample stream

CONFIGS = {
    "c1": dict(n=1_000, d=100, k=1),
    "c2": dict(n=581_012, d=54, k=2),
    "c3": dict(n=697_641, d=47_236, k=3),
    "c4": dict(n=2_396_130, d=3_231_961, k=4),
}
GEN_VERSION = 1


@dataclasses.dataclass
class Problem:
    """A CSR design matrix with +-1 labels. indices strictly increasing per row."""

    name: str
    n: int
    d: int
    indptr: np.ndarray  # int64[n+1]
    indices: np.ndarray  # int32[nnz]
    data: np.ndarray  # float64[nnz]
    y: np.ndarray  # float64[n], each +-1
    lam: float  # 1/n

    @property
    def nnz(self) -> int:
        return int(self.indptr[-1])

    def sha256(self) -> str:
        h = hashlib.sha256()
        for a in (np.asarray([self.n, self.d], dtype=np.int64), self.indptr, self.indices,
                  self.data, self.y):
            h.update(np.ascontiguousarray(a).tobytes())
        return h.hexdigest()

    def row_lengths(self) -> np.ndarray:
        return np.diff(self.indptr)

    def subset_rows(self, rows: np.ndarray, name: str | None = None) -> "Problem":
        """Rows ``rows`` (in that order) as a new Problem with the same d and lambda = 1/n'."""
        rows = np.asarray(rows, dtype=np.int64)
        lens = self.indptr[rows + 1] - self.indptr[rows]
        indptr = np.zeros(len(rows) + 1, dtype=np.int64)
        np.cumsum(lens, out=indptr[1:])
        take = np.concatenate([np.arange(self.indptr[r], self.indptr[r + 1]) for r in rows]) \
            if len(rows) else np.zeros(0, dtype=np.int64)
        return Problem(name or self.name + "_sub", len(rows), self.d, indptr,
                       self.indices[take].copy(), self.data[take].copy(), self.y[rows].copy(),
                       1.0 / max(len(rows), 1))


def _streams(k: int):
    ss = np.random.SeedSequence(BASE_SEED + k)
    a, b, c = ss.spawn(3)
    return (np.random.Generator(np.random.PCG64(a)), np.random.Generator(np.random.PCG64(b)),
            np.random.Generator(np.random.PCG64(c)))


def _finish(name, n, d, indptr, indices, data, k, rng_w, rng_noise) -> Problem:
    lens = np.diff(indptr)
    # unit l2 rows
    sq = np.add.reduceat(data * data, indptr[:-1]) if n else np.zeros(0)
    data = data / np.repeat(np.sqrt(sq), lens)
    w = rng_w.standard_normal(d)
    margin = np.add.reduceat(data * w[indices], indptr[:-1]) if n else np.zeros(0)
    noise = rng_noise.standard_normal(n)
    y = np.where(margin + 0.1 * noise >= 0.0, 1.0, -1.0)
    return Problem(name, n, d, indptr.astype(np.int64), indices.astype(np.int32),
                   data.astype(np.float64), y, 1.0 / n)


def _zipf_cdf(d: int, s: float) -> np.ndarray:
    w = np.arange(1, d + 1, dtype=np.float64) ** (-s)
    c = np.cumsum(w)
    return c / c[-1]


def _distinct_prefix_block(u, need, m, d, cdf):
    """One block of rows: u = their stream values (rows back to back, m[r] each), need = the
    distinct values wanted per row.  Returns (ok per row, ranks, rank_in_row, keep) for the
    block -- rows are independent, so blocks of rows may be processed separately (and
    concurrently) with the result of processing them all at once."""
    rows = np.repeat(np.arange(len(need), dtype=np.int64), m)
    ranks = np.searchsorted(cdf, u, side="right").astype(np.int64)
    np.minimum(ranks, d - 1, out=ranks)
    key = rows * d + ranks
    order = np.argsort(key, kind="stable")  # stable: stream order inside equal keys
    ks = key[order]
    first_sorted = np.ones(len(ks), dtype=bool)
    first_sorted[1:] = ks[1:] != ks[:-1]
    first = np.zeros(len(ks), dtype=bool)
    first[order] = first_sorted  # first occurrence, back in stream order
    # running count of distinct values per row, in stream order
    cnt = np.cumsum(first)
    row_start = np.concatenate([[0], np.cumsum(m)[:-1]])
    base = np.concatenate([[0], cnt])[row_start]
    rank_in_row = cnt - np.repeat(base, m)
    keep = first & (rank_in_row <= np.repeat(need, m))
    got = np.bincount(rows[keep], minlength=len(need))
    return got == need, rows, ranks, rank_in_row, keep


def _first_distinct_rows(rng, lens: np.ndarray, d: int, cdf: np.ndarray, perm: np.ndarray):
    """Per row i: the first lens[i] distinct values of an i.i.d. stream drawn from cdf.

    Each round draws a batch of 2*lens+8 stream values per unfinished row and keeps
    the first lens[i] distinct ones in stream order; a row whose batch holds fewer
    distinct values is redrawn from a fresh, twice longer stream.  Either way the
    row is the first-lens[i]-distinct prefix of an i.i.d. Zipf stream.  (A round's values
    are drawn block of rows by block of rows -- the same stream as one draw -- and the
    blocks are processed on a thread pool: the output does not depend on the blocking.)"""
    from concurrent.futures import ThreadPoolExecutor

    n = len(lens)
    indptr = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(lens, out=indptr[1:])
    out = np.empty(int(indptr[-1]), dtype=np.int64)
    todo = np.arange(n, dtype=np.int64)
    factor = 2
    block = 65536
    with ThreadPoolExecutor(max_workers=min(8, os.cpu_count() or 1)) as pool:
        while len(todo):
            need_all = lens[todo]
            m_all = factor * need_all + 8
            futs = []
            for b0 in range(0, len(todo), block):
                need, m = need_all[b0:b0 + block], m_all[b0:b0 + block]
                u = rng.random(int(m.sum()))  # consecutive draws: the same stream as one draw
                futs.append((b0, pool.submit(_distinct_prefix_block, u, need, m, d, cdf)))
            ok_all = np.zeros(len(todo), dtype=bool)
            for b0, f in futs:
                ok, rows, ranks, rank_in_row, keep = f.result()
                ok_all[b0:b0 + len(ok)] = ok
                m = m_all[b0:b0 + len(ok)]
                sel = keep & np.repeat(ok, m)
                dst_rows = todo[b0 + rows[sel]]
                out[indptr[dst_rows] + rank_in_row[sel] - 1] = ranks[sel]  # position = rank - 1
            todo = todo[~ok_all]
            factor *= 2

        cols = perm[out]

        def sort_rows(r0, r1):  # strictly increasing inside each row (rows are independent)
            a, b = int(indptr[r0]), int(indptr[r1])
            rr = np.repeat(np.arange(r0, r1, dtype=np.int64), lens[r0:r1])
            return a, (np.sort(rr * d + cols[a:b]) - rr * d).astype(np.int32)

        res = np.empty(int(indptr[-1]), dtype=np.int32)
        for a, v in pool.map(lambda r: sort_rows(r, min(n, r + block)), range(0, n, block)):
            res[a:a + len(v)] = v
    return indptr, res


def _gen_c1(n, d, k):
    rng, rng_w, rng_noise = _streams(k)
    mask = rng.random((n, d)) < 0.1
    empty = ~mask.any(axis=1)
    while empty.any():  # redraw empty rows (reading: rows are non-empty)
        mask[empty] = rng.random((int(empty.sum()), d)) < 0.1
        empty = ~mask.any(axis=1)
    vals = rng.standard_normal((n, d))
    lens = mask.sum(axis=1)
    indptr = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(lens, out=indptr[1:])
    rows, cols = np.nonzero(mask)
    return _finish("c1", n, d, indptr, cols, vals[rows, cols], k, rng_w, rng_noise)


def _gen_c2(n, d, k):
    assert d == 54
    rng, rng_w, rng_noise = _streams(k)
    cont = rng.standard_normal((n, 10))
    cat4 = rng.integers(0, 4, size=n)
    cat40 = rng.integers(0, 40, size=n)
    cols = np.empty((n, 12), dtype=np.int64)
    vals = np.empty((n, 12), dtype=np.float64)
    cols[:, :10] = np.arange(10)
    vals[:, :10] = cont
    cols[:, 10] = 10 + cat4
    cols[:, 11] = 14 + cat40
    vals[:, 10:] = 1.0
    # a N(0,1) draw of exactly 0.0 would store a zero; it has probability 0 here
    indptr = np.arange(0, 12 * n + 1, 12, dtype=np.int64)
    return _finish("c2", n, d, indptr, cols.ravel(), vals.ravel(), k, rng_w, rng_noise)


def _lognormal_lengths(rng, n, mean, sigma, lo, hi):
    ell = rng.lognormal(np.log(mean) - sigma * sigma / 2.0, sigma, size=n)
    return np.clip(np.rint(ell), lo, hi).astype(np.int64)


def _gen_zipf(name, n, d, k, mean, sigma, lo, hi, s, valfn):
    rng, rng_w, rng_noise = _streams(k)
    lens = _lognormal_lengths(rng, n, mean, sigma, lo, min(hi, d))
    perm = rng.permutation(d).astype(np.int64)
    cdf = _zipf_cdf(d, s)
    indptr, cols = _first_distinct_rows(rng, lens, d, cdf, perm)
    vals = valfn(rng, int(indptr[-1]))
    return _finish(name, n, d, indptr, cols, vals, k, rng_w, rng_noise)


def _gen_c3(n, d, k):
    return _gen_zipf("c3", n, d, k, 73.2, 0.63, 4, 1224, 1.1,
                     lambda rng, m: np.abs(rng.standard_normal(m)))


def _c4_vals(rng, m):
    real = rng.random(m) >= 0.9
    v = np.ones(m, dtype=np.float64)
    v[real] = rng.standard_normal(int(real.sum()))
    v[v == 0.0] = 1.0  # never store an explicit zero
    return v


def _gen_c4(n, d, k):
    return _gen_zipf("c4", n, d, k, 115.6, 0.26, 16, 414, 1.0, _c4_vals)


_GEN = {"c1": _gen_c1, "c2": _gen_c2, "c3": _gen_c3, "c4": _gen_c4}


def make(config: str, n_rows: int | None = None, cache: bool = True) -> Problem:
    """Generate config ``c1``..``c4`` (optionally with only ``n_rows`` rows, same d)."""
    cfg = CONFIGS[config]
    n = cfg["n"] if n_rows is None else int(n_rows)
    d = cfg["d"]
    path = None
    if cache and n >= 100_000:
        cdir = os.environ.get("ASAGA_DATAGEN_CACHE", "/tmp/asaga_datagen")
        path = os.path.join(cdir, f"{config}_n{n}_v{GEN_VERSION}.npz")
        if os.path.exists(path):
            try:
                z = np.load(path)
                return Problem(config, n, d, z["indptr"], z["indices"], z["data"], z["y"], 1.0 / n)
            except Exception:
                pass
    p = _GEN[config](n, d, cfg["k"])
    if n_rows is not None:
        p.name = f"{config}_n{n}"
    if path is not None:
        try:
            os.makedirs(os.path.dirname(path), exist_ok=True)
            tmp = path + f".{os.getpid()}.tmp.npz"
            np.savez(tmp, indptr=p.indptr, indices=p.indices, data=p.data, y=p.y)
            os.replace(tmp, path)
        except OSError:
            pass
    return p


def validate(p: Problem) -> None:
    """The CSR contract: sorted in-range indices, non-empty rows, labels +-1."""
    assert p.indptr.shape == (p.n + 1,) and p.indptr[0] == 0
    lens = np.diff(p.indptr)
    assert (lens > 0).all(), "empty row"
    assert p.indices.min() >= 0 and p.indices.max() < p.d
    first = np.ones(p.nnz, dtype=bool)
    first[p.indptr[:-1]] = False
    assert (np.diff(p.indices.astype(np.int64))[first[1:]] > 0).all(), "unsorted row"
    assert set(np.unique(p.y)).issubset({-1.0, 1.0})


def random_tiny(seed: int, n: int, d: int, density: float = 0.3, dense: bool = False,
                normalize: bool = True) -> Problem:
    """A tiny random CSR problem for unit tests (n, d small; non-empty rows)."""
    rng = np.random.Generator(np.random.PCG64(seed))
    if dense:
        mask = np.ones((n, d), dtype=bool)
    else:
        mask = rng.random((n, d)) < density
        for i in range(n):
            if not mask[i].any():
                mask[i, rng.integers(0, d)] = True
    vals = rng.standard_normal((n, d))
    vals[vals == 0.0] = 1.0
    lens = mask.sum(axis=1)
    indptr = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(lens, out=indptr[1:])
    rows, cols = np.nonzero(mask)
    data = vals[rows, cols]
    if normalize:
        sq = np.add.reduceat(data * data, indptr[:-1])
        data = data / np.repeat(np.sqrt(sq), lens)
    y = np.where(rng.random(n) < 0.5, -1.0, 1.0)
    return Problem(f"tiny{seed}", n, d, indptr, cols.astype(np.int32), data, y, 1.0 / n)


def to_dense(p: Problem) -> np.ndarray:
    A = np.zeros((p.n, p.d), dtype=np.float64)
    rows = np.repeat(np.arange(p.n), np.diff(p.indptr))
    A[rows, p.indices] = p.data
    return A
