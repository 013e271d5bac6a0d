"""Seeded input generators (no ACI arithmetic; see package docstring).

Seeding: ``np.random.default_rng(SeedSequence([cfg, stream, chi]))``
with streams 0 = input A / psi, 1 = input B, 2 = y_init, 3 = sample multi-indices.

Index conventions: local indices are 0-based; the
quantics bit sigma_1 (site 0) is the most significant bit (P:254-258,
Eq. quanticsrep); for the fused 2D grid of configs[4] the site index is
sigma = 2*x_bit + y_bit.
"""
from __future__ import annotations

from dataclasses import dataclass, field
import math

import numpy as np

CONFIG_NAMES = {
    0: "cfg0_cosine_L12",
    1: "cfg1_randomTT_L30_chi32",
    2: "cfg2_psi3_gaussians_L30",
    3: "cfg3_randomTT_L40_chi{chi}",
    4: "cfg4_planewave_L20_d4",
    5: "cfg5_fourier_complex_L30_K{chi}",
}


@dataclass
class TT:
    """A tensor train: cores[s] has shape (r_s, d_s, r_{s+1}), r_0 = r_L = 1."""
    cores: list
    meta: dict = field(default_factory=dict)

    @property
    def L(self) -> int:
        return len(self.cores)

    @property
    def d(self) -> list:
        return [int(c.shape[1]) for c in self.cores]

    @property
    def ranks(self) -> list:
        return [int(self.cores[0].shape[0])] + [int(c.shape[2]) for c in self.cores]


def _rng(cfg: int, stream: int, chi: int = 0) -> np.random.Generator:
    return np.random.default_rng(np.random.SeedSequence([cfg, stream, chi]))


def _block_sum(tts: list) -> TT:
    """Block-diagonal sum of TTs with equal L and d: rank(sum) = sum of ranks."""
    L = tts[0].L
    cores = []
    for s in range(L):
        parts = [t.cores[s] for t in tts]
        d = parts[0].shape[1]
        if L == 1:
            cores.append(sum(parts))
        elif s == 0:
            cores.append(np.concatenate(parts, axis=2))
        elif s == L - 1:
            cores.append(np.concatenate(parts, axis=0))
        else:
            rl = sum(p.shape[0] for p in parts)
            rr = sum(p.shape[2] for p in parts)
            c = np.zeros((rl, d, rr), np.result_type(*parts))
            i0 = j0 = 0
            for p in parts:
                c[i0:i0 + p.shape[0], :, j0:j0 + p.shape[2]] = p
                i0 += p.shape[0]
                j0 += p.shape[2]
            cores.append(c)
    return TT(cores)


def _rotation(t: float) -> np.ndarray:
    # row-vector rotation: (cos a, sin a) @ R(t) = (cos(a+t), sin(a+t))
    return np.array([[math.cos(t), math.sin(t)], [-math.sin(t), math.cos(t)]])


def _phase_tt(site_phases: list, phi: float, amp: float) -> TT:
    """Exact rank-2 TT of amp*cos(phi + sum_s site_phases[s][sigma_s]).

    site_phases[s] is a length-d_s array of angle increments for site s.
    """
    L = len(site_phases)
    v0 = amp * np.array([math.cos(phi), math.sin(phi)])
    cores = []
    for s, ph in enumerate(site_phases):
        d = len(ph)
        if L == 1:
            c = np.zeros((1, d, 1))
            for sg in range(d):
                c[0, sg, 0] = (v0 @ _rotation(ph[sg]))[0]
        elif s == 0:
            c = np.zeros((1, d, 2))
            for sg in range(d):
                c[0, sg, :] = v0 @ _rotation(ph[sg])
        elif s == L - 1:
            c = np.zeros((2, d, 1))
            for sg in range(d):
                c[:, sg, 0] = _rotation(ph[sg])[:, 0]
        else:
            c = np.zeros((2, d, 2))
            for sg in range(d):
                c[:, sg, :] = _rotation(ph[sg])
        cores.append(c)
    return TT(cores)


def cosine_sum_tt(L: int, ks, phis, amps) -> TT:
    """f(x) = sum_m amps[m] cos(2 pi ks[m] x + phis[m]) on x = sum_l 2^-l sigma_l (configs[0], R12)."""
    terms = []
    for k, phi, a in zip(ks, phis, amps):
        sp = [np.array([0.0, 2 * math.pi * k * 2.0 ** -(s + 1)]) for s in range(L)]
        terms.append(_phase_tt(sp, phi, a))
    tt = _block_sum(terms)
    tt.meta = {"kind": "cosine_sum", "ks": list(map(int, ks)), "phis": list(map(float, phis)),
               "amps": list(map(float, amps))}
    return tt


def plane_wave_tt(L: int, kxs, kys, phis, amps) -> TT:
    """sum_m amps[m] cos(2 pi (kx x + ky y) + phi) on the fused d=4 grid (configs[4], R15)."""
    terms = []
    for kx, ky, phi, a in zip(kxs, kys, phis, amps):
        sp = []
        for s in range(L):
            w = 2 * math.pi * 2.0 ** -(s + 1)
            sp.append(np.array([w * (kx * (sg >> 1) + ky * (sg & 1)) for sg in range(4)]))
        terms.append(_phase_tt(sp, phi, a))
    tt = _block_sum(terms)
    tt.meta = {"kind": "plane_wave", "kxs": list(map(int, kxs)), "kys": list(map(int, kys)),
               "phis": list(map(float, phis)), "amps": list(map(float, amps))}
    return tt


def random_tt(L: int, d: int, chi: int, rng: np.random.Generator) -> TT:
    """Cores iid N(0,1)/sqrt(chi*d), ranks [1, chi, ..., chi, 1] (configs[1],[3], R13)."""
    ranks = [1] + [chi] * (L - 1) + [1]
    scale = 1.0 / math.sqrt(chi * d)
    cores = [rng.standard_normal((ranks[s], d, ranks[s + 1])) * scale for s in range(L)]
    return TT(cores, {"kind": "random", "chi": chi})


def _tt_svd_vector(v: np.ndarray, nbits: int, cutoff: float) -> list:
    """Plain TT-SVD of a 2^nbits vector (MSB first), relative cutoff s_k <= cutoff*s_1 (R14)."""
    cores = []
    r = 1
    rest = v.reshape(1, -1)
    for _ in range(nbits - 1):
        M = rest.reshape(r * 2, -1)
        U, S, Vt = np.linalg.svd(M, full_matrices=False)
        keep = max(1, int(np.sum(S > cutoff * S[0])))
        cores.append(U[:, :keep].reshape(r, 2, keep))
        rest = S[:keep, None] * Vt[:keep]
        r = keep
    cores.append(rest.reshape(r, 2, 1))
    return cores


def gaussian3d_tt(nbits: int, cs, sigmas, amps, cutoff=1e-12) -> TT:
    """psi = sum_p a_p g_p(x) g_p(y) g_p(z), sequential x|y|z quantics (configs[2], R14)."""
    t = np.arange(2 ** nbits) / 2.0 ** nbits
    terms = []
    for c, sg, a in zip(cs, sigmas, amps):
        g = np.exp(-(t - c) ** 2 / (2 * sg ** 2))
        one = _tt_svd_vector(g, nbits, cutoff)
        cores = [x.copy() for x in one] + [x.copy() for x in one] + [x.copy() for x in one]
        cores[0] = cores[0] * a
        terms.append(TT(cores))
    tt = _block_sum(terms)
    tt.meta = {"kind": "gaussian3d", "cs": list(map(float, cs)), "sigmas": list(map(float, sigmas)),
               "amps": list(map(float, amps)), "nbits": nbits}
    return tt


def _tt_compress(cores: list, cutoff: float) -> list:
    """Input-construction rounding: left-to-right QR, right-to-left SVD keeping singular values
    s_k > cutoff * s_1 per bond (the R14 cutoff rule, on complex or real cores)."""
    cores = [c.copy() for c in cores]
    L = len(cores)
    for s in range(L - 1):
        r0, d, r1 = cores[s].shape
        Q, R = np.linalg.qr(cores[s].reshape(r0 * d, r1))
        cores[s] = Q.reshape(r0, d, Q.shape[1])
        nxt = cores[s + 1]
        cores[s + 1] = (R @ nxt.reshape(nxt.shape[0], -1)).reshape(R.shape[0], nxt.shape[1], nxt.shape[2])
    for s in range(L - 1, 0, -1):
        r0, d, r1 = cores[s].shape
        U, S, Vt = np.linalg.svd(cores[s].reshape(r0, d * r1), full_matrices=False)
        keep = max(1, int(np.sum(S > cutoff * S[0])))
        cores[s] = Vt[:keep].reshape(keep, d, r1)
        prv = cores[s - 1]
        cores[s - 1] = (prv.reshape(-1, prv.shape[2]) @ (U[:, :keep] * S[:keep])).reshape(prv.shape[0], prv.shape[1],
                                                                                           keep)
    return cores


def fourier_tt(L: int, coefs, cutoff: float = 1e-12, chunk: int = 64) -> TT:
    """Complex QTT of g(x) = sum_{k=0..K} coefs[k] e^{i k x} on x = sum_l 2^-l sigma_l in [0, 1)
    (P:289-293). Each e^{ikx} = prod_l e^{i k 2^-l sigma_l} is rank 1; chunks of `chunk`
    frequencies are block-summed and rounded (cutoff rule of R14), then the chunk TTs are summed
    pairwise with rounding after each sum, so every rounding sees a rank of at most twice the
    numerical rank O(sqrt K)."""
    coefs = np.asarray(coefs, dtype=np.complex128)
    K = len(coefs) - 1
    parts = []
    for k0 in range(0, K + 1, chunk):
        ks = np.arange(k0, min(K + 1, k0 + chunk))
        n = len(ks)
        cores = []
        for s in range(L):
            ph = np.exp(1j * ks * 2.0 ** -(s + 1))
            if s == 0:
                c = np.zeros((1, 2, n), np.complex128)
                c[0, 0, :] = coefs[ks]
                c[0, 1, :] = coefs[ks] * ph
            elif s == L - 1:
                c = np.zeros((n, 2, 1), np.complex128)
                c[:, 0, 0] = 1.0
                c[:, 1, 0] = ph
            else:
                c = np.zeros((n, 2, n), np.complex128)
                i = np.arange(n)
                c[i, 0, i] = 1.0
                c[i, 1, i] = ph
            cores.append(c)
        parts.append(TT(_tt_compress(cores, cutoff)))
    while len(parts) > 1:
        nxt = []
        for a in range(0, len(parts) - 1, 2):
            nxt.append(TT(_tt_compress(_block_sum([parts[a], parts[a + 1]]).cores, cutoff)))
        if len(parts) % 2:
            nxt.append(parts[-1])
        parts = nxt
    acc = parts[0]
    acc.meta = {"kind": "fourier", "coefs": coefs}
    return acc


def _bond_bound(d: list, s: int) -> int:
    """Largest possible rank of bond s-1|s of any tensor: min(prod d[:s], prod d[s:])."""
    left = int(np.prod([float(x) for x in d[:s]]))
    right = int(np.prod([float(x) for x in d[s:]]))
    return min(left, right, 1 << 30)


def random_init(inputs: list, maxrank: int, rng: np.random.Generator) -> TT:
    """y_init: bond ranks min_n chi^n_l capped at maxrank and at the full-tensor bound
    min(prod d_left, prod d_right) (R9'), iid N(0,1) entries (R9); complex inputs get
    iid N(0,1) real and imaginary parts."""
    L = inputs[0].L
    d = inputs[0].d
    ranks = [1] + [min(min(t.ranks[s] for t in inputs), maxrank, _bond_bound(d, s)) for s in range(1, L)] + [1]
    cplx = any(np.iscomplexobj(c) for t in inputs for c in t.cores)
    cores = []
    for s in range(L):
        shp = (ranks[s], d[s], ranks[s + 1])
        c = rng.standard_normal(shp)
        if cplx:
            c = c + 1j * rng.standard_normal(shp)
        cores.append(c)
    return TT(cores, {"kind": "y_init"})


def sample_indices(d: list, npts: int, rng: np.random.Generator) -> np.ndarray:
    """Uniform random full multi-indices, shape (npts, L), uint8."""
    L = len(d)
    out = np.empty((npts, L), dtype=np.uint8)
    for s in range(L):
        out[:, s] = rng.integers(0, d[s], size=npts)
    return out


def make_config(cfg: int, chi: int = 0, npts: int = 100_000) -> dict:
    """Build BASELINE.json configs[cfg] (chi selects the configs[3] sweep point)."""
    if cfg == 0:
        L = 12
        tts = []
        for stream in (0, 1):
            r = _rng(0, stream)
            ks = r.integers(1, 65, size=4)
            phis = r.uniform(0, 2 * math.pi, size=4)
            tts.append(cosine_sum_tt(L, ks, phis, [2.0 ** -(m + 1) for m in range(4)]))
        op = {"coef": [1.0], "expo": [[1, 1]]}
        tol, maxrank, sweeps = 1e-10, 64, 20
    elif cfg == 1:
        tts = [random_tt(30, 2, 32, _rng(1, 0)), random_tt(30, 2, 2, _rng(1, 1))]
        op = {"coef": [1.0], "expo": [[1, 1]]}
        tol, maxrank, sweeps = 1e-12, 64, 20
    elif cfg == 2:
        r = _rng(2, 0)
        cs = r.uniform(0.2, 0.8, size=8)
        sig = r.uniform(0.03, 0.1, size=8)
        amps = r.uniform(0.5, 1.0, size=8)
        tts = [gaussian3d_tt(10, cs, sig, amps)]
        op = {"coef": [1.0], "expo": [[3]]}
        tol, maxrank, sweeps = 1e-8, 256, 20
    elif cfg == 3:
        if chi not in (64, 128, 256) and chi <= 0:
            raise ValueError("configs[3] needs chi")
        tts = [random_tt(40, 2, chi, _rng(3, 0, chi)), random_tt(40, 2, 2, _rng(3, 1, chi))]
        op = {"coef": [1.0], "expo": [[1, 1]]}
        tol, maxrank, sweeps = 1e-10, 2 * chi, 4
    elif cfg == 4:
        L = 20
        tts = []
        for stream in (0, 1):
            r = _rng(4, stream)
            kx = r.integers(1, 257, size=64)
            ky = r.integers(1, 257, size=64)
            ph = r.uniform(0, 2 * math.pi, size=64)
            tts.append(plane_wave_tt(L, kx, ky, ph, [(m + 1) ** -2.0 for m in range(64)]))
        op = {"coef": [1.0, 1.0], "expo": [[1, 1], [2, 0]]}
        tol, maxrank, sweeps = 1e-8, 256, 8
    elif cfg == 5:
        # the paper's random Fourier series: two series with K+1 complex coefficients,
        # Re and Im iid U[0,1], normalised to sum |g_k|^2 = 1, L = 30 quantics, tau = 1e-8;
        # `chi` carries K here
        K = chi if chi > 0 else 100
        tts = []
        for stream in (0, 1):
            r = _rng(5, stream, K)
            c = r.uniform(0, 1, K + 1) + 1j * r.uniform(0, 1, K + 1)
            tts.append(fourier_tt(30, c / np.linalg.norm(c)))
        op = {"coef": [1.0], "expo": [[1, 1]]}
        tol, maxrank, sweeps = 1e-8, 256, 20
    else:
        raise ValueError(cfg)
    y_init = random_init(tts, maxrank, _rng(cfg, 2, chi))
    samples = sample_indices(tts[0].d, npts, _rng(cfg, 3, chi)) if npts else None
    name = CONFIG_NAMES[cfg].format(chi=chi)
    return {"cfg": cfg, "chi": chi, "name": name, "inputs": tts, "op": op, "tol": tol,
            "maxrank": maxrank, "max_sweeps": sweeps, "y_init": y_init, "samples": samples}
