"""Philox4x32-10 random streams and the synthetic dataset generator (oracle).

TEST INFRASTRUCTURE ONLY -- see oracle/__init__.py.

Restates, in vectorised numpy:
  * the block function            reference samplers.py:47-70
  * (seed, stream, block) address  reference samplers.py:78-92
    counter = [blk_lo, blk_hi, sid_lo, sid_hi], key = [seed_lo, seed_hi]
  * 53-bit uniforms in (0, 1]      reference samplers.py:95-101
  * Box-Muller normals             reference samplers.py:104-109
  * stream bookkeeping             reference samplers.py:122-147
    (every request consumes ceil(n/2) whole blocks)
  * random_profiles                reference model.py:224-249
  * synth_generate                 reference model.py:252-270
The profile/generator restatement is vectorised (no per-gene Python
objects) and bit-identical to the reference (pinned in tests/test_oracle.py).
"""

from __future__ import annotations

import numpy as np

MASK32 = np.uint64(0xFFFFFFFF)
PHILOX_M = (np.uint64(0xD2511F53), np.uint64(0xCD9E8D57))
PHILOX_W = (np.uint64(0x9E3779B9), np.uint64(0xBB67AE85))


def philox_block(ctr, key):
    """Philox4x32-10 over arrays of 32-bit words held in uint64.

    ctr: (..., 4), key: (..., 2). Returns (..., 4) uint64 words.
    """
    x = [np.asarray(ctr[..., i], dtype=np.uint64) for i in range(4)]
    k0 = np.asarray(key[..., 0], dtype=np.uint64)
    k1 = np.asarray(key[..., 1], dtype=np.uint64)
    for _ in range(10):
        a = PHILOX_M[0] * x[0]
        b = PHILOX_M[1] * x[2]
        x = [
            (b >> np.uint64(32)) ^ x[1] ^ k0,
            b & MASK32,
            (a >> np.uint64(32)) ^ x[3] ^ k1,
            a & MASK32,
        ]
        k0 = (k0 + PHILOX_W[0]) & MASK32
        k1 = (k1 + PHILOX_W[1]) & MASK32
    return np.stack(x, axis=-1)


def block_words(seed: int, stream: int, blocks: np.ndarray) -> np.ndarray:
    """Output words for block indices `blocks` of stream `stream` (samplers.py:78-92)."""
    blocks = np.asarray(blocks, dtype=np.uint64)
    s = np.uint64(stream & 0xFFFFFFFFFFFFFFFF)
    sd = np.uint64(seed & 0xFFFFFFFFFFFFFFFF)
    ctr = np.empty(blocks.shape + (4,), dtype=np.uint64)
    ctr[..., 0] = blocks & MASK32
    ctr[..., 1] = blocks >> np.uint64(32)
    ctr[..., 2] = s & MASK32
    ctr[..., 3] = s >> np.uint64(32)
    key = np.empty(blocks.shape + (2,), dtype=np.uint64)
    key[..., 0] = sd & MASK32
    key[..., 1] = sd >> np.uint64(32)
    return philox_block(ctr, key)


def words_to_uniforms(w: np.ndarray) -> np.ndarray:
    """Two uniforms in (0, 1] per block, interleaved (samplers.py:95-101)."""
    hi = (w[..., 0] << np.uint64(32)) | w[..., 1]
    lo = (w[..., 2] << np.uint64(32)) | w[..., 3]
    u = np.stack([hi, lo], axis=-1) >> np.uint64(11)
    return ((u.astype(np.float64) + 1.0) * (2.0 ** -53)).reshape(w.shape[:-1] + (2,))


def words_to_normals(w: np.ndarray) -> np.ndarray:
    """Box-Muller pair per block (samplers.py:104-109)."""
    u = words_to_uniforms(w)
    rad = np.sqrt(-2.0 * np.log(u[..., 0]))
    ang = 2.0 * np.pi * u[..., 1]
    return np.stack([rad * np.cos(ang), rad * np.sin(ang)], axis=-1)


class Stream:
    """Single (seed, stream_id) Philox stream with block cursor (samplers.py:122-147)."""

    def __init__(self, seed: int, stream_id: int = 0, block: int = 0):
        self.seed = int(seed)
        self.stream_id = int(stream_id)
        self.block = int(block)

    def _take(self, n: int, normal: bool) -> np.ndarray:
        nb = -(-n // 2)
        w = block_words(self.seed, self.stream_id, np.arange(self.block, self.block + nb, dtype=np.uint64))
        vals = words_to_normals(w) if normal else words_to_uniforms(w)
        self.block += nb
        return vals.reshape(-1)[:n]

    def uniforms(self, n: int) -> np.ndarray:
        return self._take(n, False)

    def normals(self, n: int) -> np.ndarray:
        return self._take(n, True)


# ---------------------------------------------------------------- linalg bits
DET_GUARD = 1e-300  # linalg.py:41


class SingularItem(ValueError):
    def __init__(self, idx):
        super().__init__(f"singular items {list(idx)}")
        self.indices = list(idx)


def inv_small(A: np.ndarray) -> np.ndarray:
    """Batched inverse with the reference's arithmetic.

    d=1: 1/a; d=2: adjugate (linalg.py:111-124); d=3: cofactor expansion along
    row 0 (linalg.py:127-153); d>=4: LAPACK LU (linalg.py:181-191).
    """
    A = np.asarray(A, dtype=np.float64)
    one = A.ndim == 2
    B = A[None] if one else A
    n = B.shape[-1]
    if n == 1:
        bad = np.abs(B[:, 0, 0]) < DET_GUARD
        if bad.any():
            raise SingularItem(np.nonzero(bad)[0])
        out = 1.0 / B
    elif n == 2:
        a, b, c, d = B[:, 0, 0], B[:, 0, 1], B[:, 1, 0], B[:, 1, 1]
        det = a * d - b * c
        bad = np.abs(det) < DET_GUARD
        if bad.any():
            raise SingularItem(np.nonzero(bad)[0])
        r = 1.0 / det
        out = np.empty_like(B)
        out[:, 0, 0], out[:, 0, 1], out[:, 1, 0], out[:, 1, 1] = d * r, -b * r, -c * r, a * r
    elif n == 3:
        m = lambda i, j: B[:, i, j]  # noqa: E731
        cof = np.empty_like(B)
        cof[:, 0, 0] = m(1, 1) * m(2, 2) - m(1, 2) * m(2, 1)
        cof[:, 0, 1] = m(1, 2) * m(2, 0) - m(1, 0) * m(2, 2)
        cof[:, 0, 2] = m(1, 0) * m(2, 1) - m(1, 1) * m(2, 0)
        det = m(0, 0) * cof[:, 0, 0] + m(0, 1) * cof[:, 0, 1] + m(0, 2) * cof[:, 0, 2]
        bad = np.abs(det) < DET_GUARD
        if bad.any():
            raise SingularItem(np.nonzero(bad)[0])
        cof[:, 1, 0] = m(0, 2) * m(2, 1) - m(0, 1) * m(2, 2)
        cof[:, 1, 1] = m(0, 0) * m(2, 2) - m(0, 2) * m(2, 0)
        cof[:, 1, 2] = m(0, 1) * m(2, 0) - m(0, 0) * m(2, 1)
        cof[:, 2, 0] = m(0, 1) * m(1, 2) - m(0, 2) * m(1, 1)
        cof[:, 2, 1] = m(0, 2) * m(1, 0) - m(0, 0) * m(1, 2)
        cof[:, 2, 2] = m(0, 0) * m(1, 1) - m(0, 1) * m(1, 0)
        r = 1.0 / det
        # out[i, j] = cof[j, i] / det  (the reference stores c_ji at (i, j))
        out = np.ascontiguousarray(np.swapaxes(cof, 1, 2)) * r[:, None, None]
    else:
        try:
            out = np.linalg.inv(B)
        except np.linalg.LinAlgError:
            bad = []
            for i in range(B.shape[0]):
                try:
                    np.linalg.inv(B[i])
                except np.linalg.LinAlgError:
                    bad.append(i)
            raise SingularItem(bad) from None
    return out[0] if one else out


def chol_lower(A: np.ndarray) -> np.ndarray:
    """Column-by-column Cholesky with the reference's operation order (linalg.py:195-235)."""
    A = np.asarray(A, dtype=np.float64)
    one = A.ndim == 2
    B = A[None] if one else A
    b, n, _ = B.shape
    L = np.zeros_like(B)
    for j in range(n):
        piv = B[:, j, j] - np.sum(L[:, j, :j] ** 2, axis=-1)
        if np.any(piv <= 0.0):
            raise SingularItem(np.nonzero(piv <= 0.0)[0])
        L[:, j, j] = np.sqrt(piv)
        if j + 1 < n:
            dots = np.einsum("bik,bk->bi", L[:, j + 1:, :j], L[:, j, :j])
            L[:, j + 1:, j] = (B[:, j + 1:, j] - dots) / L[:, j, j][:, None]
    return L[0] if one else L


# ---------------------------------------------------------------- generator
def profile_codes(stream: Stream, V: int, N: int, include_constant: bool = True) -> np.ndarray:
    """Integer profile codes exactly as random_profiles draws them (model.py:224-249)."""
    if N < 2 or N > 62:
        raise ValueError("N must be in [2, 62]")
    ncodes = 2 ** N
    got = []
    have = 0
    while have < V:
        u = stream.uniforms(V - have)
        c = np.minimum((u * ncodes).astype(np.int64), ncodes - 1)
        if not include_constant:
            c = c[(c != 0) & (c != ncodes - 1)]
        got.append(c)
        have += c.shape[0]
    return np.concatenate(got)[:V]


def codes_to_working(codes: np.ndarray, N: int):
    """(mu, D) of the working transform for binary codes (model.py:174-189).

    bit k of the code is network k+1's activity (model.py:247); mu = d_N and
    D_j = d_j - d_N.
    """
    bits = ((codes[:, None] >> np.arange(N, dtype=np.int64)) & 1).astype(np.float64)
    mu = bits[:, -1].copy()
    D = bits[:, :-1] - mu[:, None]
    return mu, D


def synth(stream: Stream, K, Lam, rho: float, mu: np.ndarray, D: np.ndarray) -> np.ndarray:
    """Readings r for given working profiles (model.py:252-270)."""
    K = np.atleast_1d(np.asarray(K, dtype=np.float64))
    V, dim = D.shape
    L = chol_lower(inv_small(np.atleast_2d(Lam)))
    z = stream.normals(V * dim).reshape(V, dim)
    beta = K + z @ L.T
    eps = stream.normals(V) / np.sqrt(rho)
    return np.einsum("vd,vd->v", D, beta) + mu + eps


def generate(seed: int, V: int, N: int, K, Lam, rho: float, include_constant: bool = True):
    """(r, mu, D) bit-identical to random_profiles + synth_generate on RngStream(seed)."""
    s = Stream(seed)
    codes = profile_codes(s, V, N, include_constant)
    mu, D = codes_to_working(codes, N)
    r = synth(s, K, Lam, rho, mu, D)
    return r, mu, D


def generate_slice(seed: int, lo: int, hi: int, V_total: int, N: int, K, Lam, rho: float):
    """Genes [lo, hi) of generate(seed, V_total, N, K, Lam, rho) without drawing the rest of
    the stream (include_constant=True, where every uniform is one gene): the stream is
    uniforms(V_total), normals(V_total d), normals(V_total) (model.py:224-270), each draw
    block holding two values, so a slice starting at an even gene (lo d even) begins on a
    block boundary of all three segments."""
    if lo % 2 or hi < lo or hi > V_total:
        raise ValueError("slice must start at an even gene inside the dataset")
    K = np.atleast_1d(np.asarray(K, dtype=np.float64))
    d = N - 1
    n = hi - lo
    b_z = -(-V_total // 2)
    b_e = b_z + -(-(V_total * d) // 2)
    codes = np.minimum((Stream(seed, block=lo // 2).uniforms(n) * 2 ** N).astype(np.int64), 2 ** N - 1)
    mu, D = codes_to_working(codes, N)
    L = chol_lower(inv_small(np.atleast_2d(Lam)))
    z = Stream(seed, block=b_z + lo * d // 2).normals(n * d).reshape(n, d)
    beta = K + z @ L.T
    eps = Stream(seed, block=b_e + lo // 2).normals(n) / np.sqrt(rho)
    r = np.einsum("vd,vd->v", D, beta) + mu + eps
    return r, mu, D


def make_regime(V: int, seed: int = 0, N: int = 3, K=None, rho: float = 100.0, include_constant=True):
    """The reference test-suite regime (reference tests/conftest.py:15-26).

    N=3: K=(0.1, 0.3), Lambda = inv([[0.01, 0.005], [0.005, 0.008]]);
    otherwise K = 0.2 everywhere, Lambda = inv(0.01 I) = 100 I.
    Returns (r, mu, D, K, Lam).
    """
    if N == 3:
        lam = np.linalg.inv(np.array([[0.01, 0.005], [0.005, 0.008]]))
        K = np.array([0.1, 0.3]) if K is None else np.asarray(K, dtype=float)
    else:
        lam = np.linalg.inv(0.01 * np.eye(N - 1))
        if K is None or len(K) != N - 1:
            K = np.full(N - 1, 0.2)
    r, mu, D = generate(seed, V, N, K, lam, rho, include_constant)
    return r, mu, D, np.asarray(K, dtype=float), lam
