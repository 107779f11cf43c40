"""CPU oracle for the NDF hot path -- TEST INFRASTRUCTURE ONLY.

This module is a plain-NumPy restatement of the reference algorithms on the
hot path (``/root/reference/pkg/src/ndf``).  It is the *checker*: only
``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline /
reference arm may import it.  The product package
(``paper_2307_02203_b200``) never imports it and has no CPU fallback.

Every function cites the reference ``file:line`` it restates and follows the
reference's operation order so that results agree bit for bit wherever the
reference's arithmetic is deterministic (fp64 embedding, ``einsum`` matmul,
KSG counts).  Where BASELINE.json asks for architecture the reference cannot
express (dense anisotropic latent grid, ``sum_absdiff``
merge, SiLU, tanh/softplus heads) the restatement extends the reference's own
code path in the same style; parity for those deltas is pinned only by this
restatement ("parity unpinned by reference tests" for those pieces, see
DESIGN.md).

Pinning: ``tests/test_oracle.py`` checks this module against golden vectors
produced by importing the unmodified reference (``tests/golden/make_golden.py``)
and against the reference's own known-answer tests.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

# reference: pkg/src/ndf/measures.py:33
JITTER_SEED = 0x5D17E3
# reference: pkg/src/ndf/encoding.py:19, pkg/src/ndf/ensemble.py:31
NODE_SNAP = 1e-9


# ---------------------------------------------------------------------------
# positions and encoders


def grid_positions(dims):
    """measures.py:240-252 -- node coordinates in Omega, x fastest."""
    def axis(n):
        if n == 1:
            return np.zeros(1)
        return 2.0 * np.arange(n) / (n - 1) - 1.0

    x, y, z = dims
    zz, yy, xx = np.meshgrid(axis(z), axis(y), axis(x), indexing="ij")
    return np.column_stack([xx.ravel(), yy.ravel(), zz.ravel()])


def grid_positions_of(dims, vertices):
    """Rows ``vertices`` of grid_positions(dims), without materialising the grid
    (same per-axis formula, so the same bits)."""
    def axis(n):
        if n == 1:
            return np.zeros(1)
        return 2.0 * np.arange(n) / (n - 1) - 1.0

    x, y, z = dims
    v = np.asarray(vertices, dtype=np.int64)
    ix, iy, iz = v % x, (v // x) % y, v // (x * y)
    return np.column_stack([axis(x)[ix], axis(y)[iy], axis(z)[iz]])


def fourier_encode(positions, L):
    """encoding.py:37-51 -- octave-major, axis-minor, sin before cos."""
    pos = np.atleast_2d(np.asarray(positions, dtype=np.float64))
    out = np.empty((pos.shape[0], 6 * L))
    for i in range(L):
        phase = (2.0 ** i * np.pi) * pos
        out[:, 6 * i + 0:6 * i + 6:2] = np.sin(phase)
        out[:, 6 * i + 1:6 * i + 6:2] = np.cos(phase)
    return out


def level_coords(p, res):
    """encoding.py:105-113 (also ensemble.py:115-127) -- base index + weight."""
    u = (np.clip(p, -1.0, 1.0) + 1.0) * 0.5 * (res - 1)
    i0 = np.floor(u).astype(np.int64)
    np.clip(i0, 0, res - 2, out=i0)
    t = u - i0
    t[t < NODE_SNAP] = 0.0
    t[t > 1.0 - NODE_SNAP] = 1.0
    return i0, t


# encoding.py:116-118 -- dx fastest, then dy, then dz
CORNER_OFFSETS = np.array([(dx, dy, dz)
                           for dz in (0, 1) for dy in (0, 1) for dx in (0, 1)],
                          dtype=np.int64)


def dense_grid_encode(positions, table):
    """Dense anisotropic latent grid, restating HashGrid.encode's dense branch.

    ``table`` is (rz, ry, rx, C) fp32.  Follows encoding.py:149-178 with a
    per-axis resolution: per-axis ``level_coords`` (encoding.py:105-113),
    dense index ``ix + rx*(iy + ry*iz)`` (encoding.py:97-98 with per-axis
    strides), weights built as ``w = ((1*wx)*wy)*wz`` (encoding.py:156-160)
    and the fp64 corner sum in corner order (``einsum "mc,mcf->mf"``,
    encoding.py:176).
    """
    pos = np.atleast_2d(np.asarray(positions, dtype=np.float64))
    rz, ry, rx, C = table.shape
    flat = table.reshape(rz * ry * rx, C).astype(np.float64)
    i0 = np.empty((pos.shape[0], 3), dtype=np.int64)
    t = np.empty((pos.shape[0], 3))
    for axis, res in enumerate((rx, ry, rz)):
        i0[:, axis], t[:, axis] = level_coords(pos[:, axis], res)
    corners = i0[:, None, :] + CORNER_OFFSETS[None, :, :]
    idx = corners[..., 0] + rx * (corners[..., 1] + ry * corners[..., 2])
    w = np.ones(corners.shape[:2])
    for axis in range(3):
        frac = t[:, axis:axis + 1]
        on = CORNER_OFFSETS[:, axis][None, :]
        w = w * np.where(on, frac, 1.0 - frac)
    feats = flat[idx]
    return np.einsum("mc,mcf->mf", w, feats, optimize=False)


HASH_PRIMES = (np.uint64(1), np.uint64(2654435761), np.uint64(805459861))   # encoding.py:17


@dataclass
class HashGridSpec:
    """The reference HashGrid (encoding.py:55-86): tables (levels, 2^T, F)."""

    tables: np.ndarray
    level_res: tuple          # round(base * growth^l) (encoding.py:82-83)
    log2_table: int


def hash_grid_encode(positions, grid: HashGridSpec):
    """HashGrid.encode (encoding.py:163-178) via _level_lookup (:149-161): per level,
    level_coords, corner rows dense (res^3 <= 2^T) or XOR-prime hashed mod 2^T
    (_corner_indices, :90-102), weights ((1*wx)*wy)*wz, fp64 corner sum."""
    pos = np.atleast_2d(np.asarray(positions, dtype=np.float64))
    levels, T, F = grid.tables.shape
    out = np.empty((pos.shape[0], levels * F))
    for lv in range(levels):
        res = grid.level_res[lv]
        i0 = np.empty((pos.shape[0], 3), dtype=np.int64)
        t = np.empty((pos.shape[0], 3))
        for axis in range(3):
            i0[:, axis], t[:, axis] = level_coords(pos[:, axis], res)
        corners = i0[:, None, :] + CORNER_OFFSETS[None, :, :]
        ix, iy, iz = corners[..., 0], corners[..., 1], corners[..., 2]
        if res ** 3 <= T:
            idx = (ix + res * (iy + res * iz)).astype(np.int64)
        else:
            h = (ix.astype(np.uint64) * HASH_PRIMES[0] ^ iy.astype(np.uint64) * HASH_PRIMES[1]
                 ^ iz.astype(np.uint64) * HASH_PRIMES[2])
            idx = (h & np.uint64(T - 1)).astype(np.int64)
        w = np.ones(corners.shape[:2])
        for axis in range(3):
            frac = t[:, axis:axis + 1]
            on = CORNER_OFFSETS[:, axis][None, :]
            w = w * np.where(on, frac, 1.0 - frac)
        feats = grid.tables[lv].astype(np.float64)[idx]
        out[:, lv * F:(lv + 1) * F] = np.einsum("mc,mcf->mf", w, feats, optimize=False)
    return out


def embed(positions, table, L):
    """model.py:169-177 -- [raw | fourier | grid] computed in fp64, cast fp32.
    ``table``: dense (rz, ry, rx, C) array or a HashGridSpec (reference family)."""
    pos = np.atleast_2d(np.asarray(positions, dtype=np.float64))
    clamped = np.clip(pos, -1.0, 1.0)
    grid = (hash_grid_encode(clamped, table) if isinstance(table, HashGridSpec)
            else dense_grid_encode(clamped, table))
    parts = [clamped, fourier_encode(clamped, L), grid]
    return np.concatenate(parts, axis=1).astype(np.float32)


# ---------------------------------------------------------------------------
# merge, activations, MLP


def merge(mode, a, b):
    """model.py:279-286 plus BASELINE's ``sum_absdiff`` = [a+b, |a-b|]."""
    if mode == "multiply":
        return a * b
    if mode == "concat":
        return np.concatenate([a, b], axis=1)
    if mode == "add":
        return a + b
    if mode == "absdiff":
        return np.abs(a - b)
    if mode == "sum_absdiff":
        return np.concatenate([a + b, np.abs(a - b)], axis=1)
    raise ValueError(mode)


def activation(kind, x):
    """nn.py:23-32 plus SiLU (BASELINE), evaluated in the input dtype."""
    x = np.asarray(x)
    if kind == "relu":
        return np.maximum(x, x.dtype.type(0))
    if kind == "snake":                                   # nn.py:28-29
        return x + np.sin(x) ** 2
    if kind == "snake_alt":
        one = x.dtype.type(1)
        return x.dtype.type(0.5) * (x + one - np.cos(x.dtype.type(2) * x))
    if kind == "silu":
        return x / (x.dtype.type(1) + np.exp(-x))
    raise ValueError(kind)


def head(kind, z):
    """Output head (BASELINE delta): linear (reference, nn.py:136), tanh, softplus."""
    z = np.asarray(z)
    if kind == "linear":
        return z
    if kind == "tanh":
        return np.tanh(z)
    if kind == "softplus":
        return np.maximum(z, z.dtype.type(0)) + np.log1p(np.exp(-np.abs(z)))
    raise ValueError(kind)


def matmul_exact(a, b):
    """nn.py:18-20 -- einsum without optimisation (sequential fp32 k-sum)."""
    return np.einsum("ij,jk->ik", a, b, optimize=False)


def mlp_forward(weights, biases, act, x):
    """nn.py:124-137 -- affine + activation per hidden layer, affine output."""
    h = np.atleast_2d(x)
    last = len(weights) - 1
    for i, (w, b) in enumerate(zip(weights, biases)):
        z = matmul_exact(h, w) + b
        h = z if i == last else activation(act, z)
    return h


# ---------------------------------------------------------------------------
# model


@dataclass
class OracleModel:
    """NDF of either family: BASELINE (dense latent grid, no encoder MLP) or the
    reference's own (HashGridSpec grids + per-branch encoder MLPs, model.py:105-189)."""

    L: int
    grid_mu: object              # (rz, ry, rx, C) fp32 array, or HashGridSpec
    grid_nu: object
    weights: list = field(default_factory=list)   # decoder (fan_in, fan_out) fp32
    biases: list = field(default_factory=list)
    merge: str = "sum_absdiff"
    act: str = "silu"
    head: str = "tanh"
    enc_mu: tuple = ((), ())     # encoder (weights, biases); empty = identity (nn.py:84-86)
    enc_nu: tuple = ((), ())

    def encode(self, positions, grid, enc):
        """embed, then the branch encoder MLP (model.py:184-185)."""
        e = embed(positions, grid, self.L)
        ws, bs = enc
        return mlp_forward(list(ws), list(bs), self.act, e) if len(ws) else e

    def forward(self, p_mu, p_nu):
        """model.py:179-189."""
        a = self.encode(p_mu, self.grid_mu, self.enc_mu)
        b = self.encode(p_nu, self.grid_nu, self.enc_nu)
        if a.shape[0] == 1 and b.shape[0] > 1:
            a = np.broadcast_to(a, b.shape)
        if b.shape[0] == 1 and a.shape[0] > 1:
            b = np.broadcast_to(b, a.shape)
        z = mlp_forward(self.weights, self.biases, self.act, merge(self.merge, a, b))
        return head(self.head, z)[:, 0]


def latent_resolution(dims, factor):
    """per-axis r_a = max(2, ceil(n_a / f))."""
    return tuple(max(2, -(-int(n) // int(factor))) for n in dims)


def build_model(dims, factor=8, channels=16, L=6, hidden=128, decoder_layers=4,
                merge_mode="sum_absdiff", act="silu", head_kind="tanh", seed=0,
                grid_scale=1e-4, shared=True):
    """Seeded weights in the reference's RNG order (model.py:131-142).

    grid_mu <- uniform(-s, s) (encoding.py:139-147, s=1e-4 in the reference),
    encoders are identities (no draws, nn.py:84-86), optional grid_nu, then
    decoder Kaiming-uniform fan-in with zero biases (nn.py:76-93).
    """
    rng = np.random.default_rng(seed)
    rx, ry, rz = latent_resolution(dims, factor)
    grid_mu = rng.uniform(-grid_scale, grid_scale, size=(rz, ry, rx, channels)).astype(np.float32)
    grid_nu = grid_mu if shared else rng.uniform(
        -grid_scale, grid_scale, size=(rz, ry, rx, channels)).astype(np.float32)
    E = 3 + 6 * L + channels
    din = 2 * E if merge_mode in ("sum_absdiff", "concat") else E
    widths = [din] + [hidden] * (decoder_layers - 1) + [1]
    ws, bs = [], []
    for fan_in, fan_out in zip(widths[:-1], widths[1:]):
        bound = np.sqrt(6.0 / fan_in)
        ws.append(rng.uniform(-bound, bound, (fan_in, fan_out)).astype(np.float32))
        bs.append(np.zeros(fan_out, dtype=np.float32))
    return OracleModel(L, grid_mu, grid_nu, ws, bs, merge_mode, act, head_kind)


def reconstruct_field(model: OracleModel, ref, dims, role="reference-is-mu",
                      batch_size=65536, clamp=False, vertices=None):
    """service.py:46-84 -- ref embedded once, query grid in batches.

    ``vertices`` (optional flat indices) restricts evaluation to a subset of
    the grid nodes (used for bounded CPU samples); results per vertex are
    identical to the full evaluation because per-row arithmetic does not
    depend on the batch layout (nn.py:1-7).
    """
    ref = np.asarray(ref, dtype=np.float64).reshape(1, 3)
    if vertices is not None:
        positions = grid_positions_of(dims, vertices)
    else:
        positions = grid_positions(dims)
    ref_is_mu = role == "reference-is-mu"
    ref_grid = model.grid_mu if ref_is_mu else model.grid_nu
    query_grid = model.grid_nu if ref_is_mu else model.grid_mu
    ref_enc = model.enc_mu if ref_is_mu else model.enc_nu
    query_enc = model.enc_nu if ref_is_mu else model.enc_mu
    ref_features = model.encode(ref, ref_grid, ref_enc)
    out = np.empty(positions.shape[0], dtype=np.float32)
    for s in range(0, positions.shape[0], batch_size):
        q = model.encode(positions[s:s + batch_size], query_grid, query_enc)
        r = np.broadcast_to(ref_features, q.shape)
        merged = merge(model.merge, r, q) if ref_is_mu else merge(model.merge, q, r)
        z = mlp_forward(model.weights, model.biases, model.act, merged)
        out[s:s + batch_size] = head(model.head, z)[:, 0]
    if clamp:
        np.clip(out, -1.0, 1.0, out=out)
    return out


# ---------------------------------------------------------------------------
# ensemble sampling


def fractional_index(p, n):
    """ensemble.py:115-127."""
    return level_coords(p, n)


def sample_many(grids, positions, chunk=8192):
    """ensemble.py:130-167 -- fp64 trilinear over all members.

    ``grids`` is one variable's (N, nz, ny, nx) fp32 block.
    """
    N, nz, ny, nx = grids.shape
    pos = np.atleast_2d(np.asarray(positions, dtype=np.float64))
    out = np.empty((pos.shape[0], N), dtype=np.float64)
    for s in range(0, pos.shape[0], chunk):
        block = pos[s:s + chunk]
        ix, tx = fractional_index(block[:, 0], nx)
        iy, ty = fractional_index(block[:, 1], ny)
        iz, tz = fractional_index(block[:, 2], nz)
        acc = np.zeros((block.shape[0], N), dtype=np.float64)
        for dz in (0, 1):
            wz = tz if dz else 1.0 - tz
            for dy in (0, 1):
                wy = ty if dy else 1.0 - ty
                for dx in (0, 1):
                    wx = tx if dx else 1.0 - tx
                    w = wz * wy * wx
                    corner = grids[:, iz + dz, iy + dy, ix + dx]
                    acc += w[:, None] * corner.T
        out[s:s + chunk] = acc
    return out


# ---------------------------------------------------------------------------
# estimators


def pearson(a, b):
    """measures.py:59-81 (returns None where the reference raises)."""
    a = np.asarray(a, dtype=np.float64).ravel()
    b = np.asarray(b, dtype=np.float64).ravel()
    ac = a - a.mean()
    bc = b - b.mean()
    var_a = float(ac @ ac)
    var_b = float(bc @ bc)
    if var_a == 0.0 or var_b == 0.0:
        return None
    if np.array_equal(a, b):
        return 1.0
    r = float(ac @ bc) / np.sqrt(var_a * var_b)
    return float(min(1.0, max(-1.0, r)))


def pearson_against(ref, samples):
    """measures.py:84-108 -- NaN for degenerate rows, self rows -> 1.0."""
    ref = np.asarray(ref, dtype=np.float64).ravel()
    samples = np.asarray(samples, dtype=np.float64)
    rc = ref - ref.mean()
    var_ref = float(rc @ rc)
    out = np.full(samples.shape[0], np.nan)
    if var_ref == 0.0:
        return out
    sc = samples - samples.mean(axis=1, keepdims=True)
    var_s = np.einsum("ij,ij->i", sc, sc)
    ok = var_s > 0.0
    out[ok] = (sc[ok] @ rc) / np.sqrt(var_s[ok] * var_ref)
    np.clip(out, -1.0, 1.0, out=out)
    near = np.flatnonzero(ok & (out > 1.0 - 1e-9))
    for i in near:
        if np.array_equal(samples[i], ref):
            out[i] = 1.0
    return out


def pearson_rowwise(a, b):
    """measures.py:111-133."""
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    ac = a - a.mean(axis=1, keepdims=True)
    bc = b - b.mean(axis=1, keepdims=True)
    var_a = np.einsum("ij,ij->i", ac, ac)
    var_b = np.einsum("ij,ij->i", bc, bc)
    out = np.full(a.shape[0], np.nan)
    ok = (var_a > 0.0) & (var_b > 0.0)
    out[ok] = (np.einsum("ij,ij->i", ac, bc)[ok] / np.sqrt(var_a[ok] * var_b[ok]))
    np.clip(out, -1.0, 1.0, out=out)
    same = ok & (out > 1.0 - 1e-9)
    for i in np.flatnonzero(same):
        if np.array_equal(a[i], b[i]):
            out[i] = 1.0
    return out


def digamma(x):
    """measures.py:136-165 -- recurrence shift + asymptotic series (fp64)."""
    x = np.asarray(x, dtype=np.float64)
    scalar = x.ndim == 0
    x = np.atleast_1d(x).copy()
    acc = np.zeros_like(x)
    for _ in range(10):
        small = x < 10.0
        if not small.any():
            break
        acc[small] -= 1.0 / x[small]
        x[small] += 1.0
    inv2 = 1.0 / (x * x)
    series = (np.log(x) - 0.5 / x
              - inv2 * (1.0 / 12.0 - inv2 * (1.0 / 120.0 - inv2 * (
                  1.0 / 252.0 - inv2 * (1.0 / 240.0 - inv2 / 132.0)))))
    out = acc + series
    return float(out[0]) if scalar else out


def tie_jitter(n):
    """measures.py:168-170."""
    return np.random.default_rng(JITTER_SEED).random(n) - 0.5


def jitter(v, r):
    """measures.py:190-192 -- v + r*(1e-10*ptp(v)) in fp64."""
    v = np.asarray(v, dtype=np.float64).ravel()
    return v + r * (1e-10 * np.ptp(v))


def ksg_counts_bruteforce(a, b, k):
    """measures.py:183-201 restated in brute force (what the GPU kernel computes).

    eps_i = k-th smallest max-norm distance over j != i (the cKDTree query
    of k+1 neighbours including self, measures.py:193-195);
    n_x = #{j : fl(a_i - eps) < a_j < fl(a_i + eps)} - 1 (measures.py:198-201).
    Returns (eps, n_x, n_y) on the jittered inputs.
    """
    n = a.size
    r = tie_jitter(n)
    aj = jitter(a, r)
    bj = jitter(b, r)
    eps = np.empty(n)
    for s in range(0, n, 256):
        da = np.abs(aj[s:s + 256, None] - aj[None, :])
        db = np.abs(bj[s:s + 256, None] - bj[None, :])
        d = np.maximum(da, db)
        d[np.arange(d.shape[0]), np.arange(s, s + d.shape[0])] = np.inf
        eps[s:s + 256] = np.partition(d, k - 1, axis=1)[:, k - 1]
    sa = np.sort(aj)
    sb = np.sort(bj)
    n_x = (np.searchsorted(sa, aj + eps, "left") - np.searchsorted(sa, aj - eps, "right") - 1)
    n_y = (np.searchsorted(sb, bj + eps, "left") - np.searchsorted(sb, bj - eps, "right") - 1)
    return eps, n_x, n_y


def ksg_counts_kdtree(a, b, k):
    """measures.py:183-201 exactly as the reference (scipy cKDTree, pinned
    third-party dependency scipy==1.18.1 ``cKDTree.query(k+1, p=inf)``)."""
    from scipy.spatial import cKDTree
    n = a.size
    r = tie_jitter(n)
    aj = jitter(a, r)
    bj = jitter(b, r)
    tree = cKDTree(np.column_stack([aj, bj]))
    dist, _ = tree.query(np.column_stack([aj, bj]), k=k + 1, p=np.inf)
    eps = dist[:, k]
    sa = np.sort(aj)
    sb = np.sort(bj)
    n_x = (np.searchsorted(sa, aj + eps, "left") - np.searchsorted(sa, aj - eps, "right") - 1)
    n_y = (np.searchsorted(sb, bj + eps, "left") - np.searchsorted(sb, bj - eps, "right") - 1)
    return eps, n_x, n_y


def ksg_from_counts(n_x, n_y, k):
    """measures.py:202-203 -- psi(k) + psi(N) - mean(psi(n_x+1) + psi(n_y+1))."""
    n = n_x.size
    if np.any(n_x + 1.0 <= 0.0) or np.any(n_y + 1.0 <= 0.0):
        return None   # the reference's digamma raises ParameterError here
    point_terms = digamma(n_x + 1.0) + digamma(n_y + 1.0)
    return float(digamma(float(k)) + digamma(float(n)) - np.mean(point_terms))


def ksg_mi(a, b, k=3, counts="kdtree"):
    """measures.py:173-203."""
    a = np.asarray(a, dtype=np.float64).ravel()
    b = np.asarray(b, dtype=np.float64).ravel()
    fn = ksg_counts_kdtree if counts == "kdtree" else ksg_counts_bruteforce
    _, n_x, n_y = fn(a, b, k)
    return ksg_from_counts(n_x, n_y, k)


def ground_truth_field(grids, measure, ref, dims, k=3, chunk=4096, vertices=None):
    """measures.py:273-315 for one variable (var_mu == var_nu).

    ``grids`` is (N, nz, ny, nx) fp32.  ``vertices`` optionally restricts the
    evaluation to a subset of flat grid indices (bounded CPU samples).
    """
    if vertices is not None:
        positions = grid_positions_of(dims, vertices)
    else:
        positions = grid_positions(dims)
    ref = np.asarray(ref, dtype=np.float64).reshape(3)
    ref_vec = sample_many(grids, ref.reshape(1, 3))[0]
    if measure == "pearson":
        out = np.empty(positions.shape[0])
        for s in range(0, positions.shape[0], chunk):
            block = sample_many(grids, positions[s:s + chunk])
            out[s:s + chunk] = pearson_against(ref_vec, block)
        out[np.isnan(out)] = 0.0
    else:
        parts = []
        for s in range(0, positions.shape[0], chunk):
            samples = sample_many(grids, positions[s:s + chunk])
            parts.append(np.array([ksg_mi(ref_vec, row, k) for row in samples]))
        out = np.concatenate(parts) if parts else np.empty(0)
    return out.astype(np.float32)


# ---------------------------------------------------------------------------
# synthetic ensembles (BASELINE generator; numpy backend for CPU configs)


def synthetic_member_noise(rng, dims, count, lengths):
    """FFT-filtered white noise, amplitude exp(-l^2 k^2 / 4) per axis."""
    nx, ny, nz = dims
    noise = rng.standard_normal((count, nz, ny, nx))
    spec = np.fft.rfftn(noise, axes=(1, 2, 3))
    kz = 2 * np.pi * np.fft.fftfreq(nz)
    ky = 2 * np.pi * np.fft.fftfreq(ny)
    kx = 2 * np.pi * np.fft.rfftfreq(nx)
    lx, ly, lz = lengths
    filt = (np.exp(-(lz * kz[:, None, None]) ** 2 / 4)
            * np.exp(-(ly * ky[None, :, None]) ** 2 / 4)
            * np.exp(-(lx * kx[None, None, :]) ** 2 / 4))
    return np.fft.irfftn(spec * filt, s=(nz, ny, nx), axes=(1, 2, 3))
