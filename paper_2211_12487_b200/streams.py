"""Seeded synthetic increment streams for BASELINE.json configs 0-4.

The paper's datasets (ATARI frames, gel simulations)
are not available, so these seeded generators with the configs' shapes,
sizes and value distributions stand in for them.  Every choice BASELINE
leaves open is fixed here and recorded in DESIGN.md §6:

* cfg0  random TT, ranks (1,3,3,3,3) (r_4 := 3), QR-orthonormal N(0,1) cores,
        N(0,1) coefficients, N(0,1) noise at 1 % of the signal norm.
* cfg1  video-like 210x160x3 -> (14,15,16,10,3); 20 separable cosine modes
        (frequency ~ U(0.5, 4) cycles per axis, phase ~ U(0, 2pi), channel
        weights ~ N(0,1)), amplitudes ~ N(0,1) redrawn per frame, +2 modes
        every 5 increments, 2 % noise.
* cfg2  simulation-like 64^3 x 3 -> (8,8,8,8,8,8,3); complex Fourier modes
        with |k|_2 <= 6 per component, coefficients an AR(1) process
        (rho = 0.95, unit variance per real/imaginary part) over snapshots,
        0.5 % noise.
* cfg3  random TT with true ranks 12 per bond (r_1 capped to 8); odd
        increments re-sample coefficients inside the span seen so far (skip
        path); even increments k >= 2 add one new rank-1 drift direction with
        amplitude 0.3*sqrt(12)*N(0,1) per observation; 0.1 % noise.
* cfg4  cfg3 generator with batch 2048 (sharded over GPUs by the bench).

Seeds are counter-based (``numpy.random.default_rng([seed, stream, k])``),
so increment k can be regenerated independently (cfg2's AR(1) state is the
exception and is advanced sequentially).  Layout: first-index-fastest numpy
arrays of shape ``modes + (batch,)``.

``DeviceStream`` produces the same distributions directly in HBM (torch on
CUDA) for the benchmark; it is input synthesis, not part of the product path.
"""
from __future__ import annotations

import math
from dataclasses import dataclass
from typing import List, Optional, Sequence, Tuple

import numpy as np


@dataclass(frozen=True)
class StreamConfig:
    name: str
    modes: Tuple[int, ...]
    batch: int
    increments: int
    eps: float
    kind: str


CONFIGS = {
    0: StreamConfig("cfg0-random-tt", (8, 8, 8, 8), 1, 64, 0.1, "random_tt"),
    1: StreamConfig("cfg1-video", (14, 15, 16, 10, 3), 100, 40, 0.1, "video"),
    2: StreamConfig("cfg2-simulation", (8, 8, 8, 8, 8, 8, 3), 32, 50, 0.05, "simulation"),
    3: StreamConfig("cfg3-ttice-star", (8,) * 7, 256, 30, 0.01, "drift_tt"),
    4: StreamConfig("cfg4-scaling", (8,) * 7, 2048, 30, 0.01, "drift_tt"),
}


def _orthonormal(rng: np.random.Generator, rows: int, cols: int) -> np.ndarray:
    q, _ = np.linalg.qr(rng.standard_normal((rows, cols)))
    return q


def capped_ranks(modes: Sequence[int], r: int) -> List[int]:
    """(1, r_1, ..., r_d) with r_i <= r_{i-1} n_i (orthonormal left unfoldings)."""
    ranks = [1]
    for n in modes:
        ranks.append(min(r, ranks[-1] * n))
    return ranks


def tt_chain(cores: Sequence[np.ndarray]) -> np.ndarray:
    """(prod n) x r_d basis of left-unfolding cores (spatial_chain, tensor_train.cpp:152-166)."""
    acc = cores[0]  # n_1 x r_1 (r_0 = 1)
    rows = cores[0].shape[0]
    for u in cores[1:]:
        r_prev = acc.shape[1]
        n = u.shape[0] // r_prev
        right = np.reshape(u, (r_prev, n * u.shape[1]), order="F")
        nxt = acc @ right
        rows *= n
        acc = np.reshape(nxt, (rows, u.shape[1]), order="F")
    return acc


def _add_noise(rng: np.random.Generator, s: np.ndarray, rel: float) -> np.ndarray:
    nz = rng.standard_normal(s.shape)
    ns = float(np.linalg.norm(nz))
    sn = float(np.linalg.norm(s))
    if ns > 0 and sn > 0:
        s = s + (rel * sn / ns) * nz
    return s


class Stream:
    """Host (numpy) increment stream.  ``modes``/``batch`` override the config's
    shape for scaled-down parity runs (cfg0/3/4 random-TT kinds; cfg2 takes
    ``grid``; cfg1 takes ``batch`` only)."""

    def __init__(self, cfg: int, seed: int = 0, batch: Optional[int] = None, modes: Optional[Sequence[int]] = None,
                 true_rank: Optional[int] = None, grid: int = 64, drift_amp: float = 0.3, noise: Optional[float] = None):
        self.cfg = CONFIGS[cfg]
        self.cfg_id = cfg
        self.seed = seed
        self.kind = self.cfg.kind
        self.batch = batch or self.cfg.batch
        self.eps = self.cfg.eps
        self.increments = self.cfg.increments
        self.drift_amp = drift_amp
        if self.kind in ("random_tt", "drift_tt"):
            self.modes = tuple(modes) if modes is not None else self.cfg.modes
            tr = true_rank or (3 if self.kind == "random_tt" else 12)
            self.ranks = capped_ranks(self.modes, tr)
            rng = np.random.default_rng([seed, 0])
            self.cores = [_orthonormal(rng, self.ranks[i] * n, self.ranks[i + 1]) for i, n in enumerate(self.modes)]
            self.phi = tt_chain(self.cores)
            self.noise = noise if noise is not None else (0.01 if self.kind == "random_tt" else 1e-3)
            self._drifts = {}
        elif self.kind == "video":
            self.modes = self.cfg.modes
            self.noise = noise if noise is not None else 0.02
            rng = np.random.default_rng([seed, 0])
            nmax = 20 + 2 * (self.increments // 5 + 1)
            x = np.arange(210)[None, :]
            y = np.arange(160)[None, :]
            fx, px = rng.uniform(0.5, 4.0, (nmax, 1)), rng.uniform(0, 2 * np.pi, (nmax, 1))
            fy, py = rng.uniform(0.5, 4.0, (nmax, 1)), rng.uniform(0, 2 * np.pi, (nmax, 1))
            self.prof_x = np.cos(2 * np.pi * fx * x / 210.0 + px)
            self.prof_y = np.cos(2 * np.pi * fy * y / 160.0 + py)
            self.prof_c = rng.standard_normal((nmax, 3))
        elif self.kind == "simulation":
            if grid % 8 and grid != 16:
                raise ValueError("grid must split into two equal factors")
            h = int(round(math.sqrt(grid)))
            if h * h != grid:
                raise ValueError("grid must be a perfect square (64 -> 8x8, 16 -> 4x4)")
            self.grid = grid
            self.modes = (h, h, h, h, h, h, 3)
            self.noise = noise if noise is not None else 5e-3
            kr = np.arange(-6, 7)
            kk = np.array([(a, b, c) for a in kr for b in kr for c in kr if a * a + b * b + c * c <= 36])
            self.kvec = kk
            self.kidx = tuple((kk % grid).T)
            self._ar_t = 0
            self._ar_state = None
            self._ar_rng = np.random.default_rng([seed, 2])
        else:
            raise ValueError(self.kind)

    # -- drift directions (cfg3/cfg4): rank-1 unit tensors
    def drift(self, k: int) -> np.ndarray:
        if k not in self._drifts:
            rng = np.random.default_rng([self.seed, 3, k])
            v = np.ones(1)
            for n in self.modes:  # first-index-fastest: kron(v_last, ..., v_1)
                u = rng.standard_normal(n)
                u /= np.linalg.norm(u)
                v = np.kron(u, v)
            self._drifts[k] = v
        return self._drifts[k]

    def drift_ids(self, k: int) -> List[int]:
        """Drift directions present in increment k (new ones at even k >= 2)."""
        return [j for j in range(2, k + 1, 2)]

    def is_redundant(self, k: int) -> bool:
        return self.kind == "drift_tt" and k % 2 == 1

    def increment(self, k: int, batch: Optional[int] = None) -> np.ndarray:
        b = batch or self.batch
        g = np.random.default_rng([self.seed, 1, k])
        if self.kind == "random_tt":
            c = g.standard_normal((self.phi.shape[1], b))
            s = self.phi @ c
        elif self.kind == "drift_tt":
            c = g.standard_normal((self.phi.shape[1], b))
            s = self.phi @ c
            ids = self.drift_ids(k)
            if ids:
                amp = self.drift_amp * math.sqrt(self.phi.shape[1])
                cd = amp * g.standard_normal((len(ids), b))
                dm = np.stack([self.drift(j) for j in ids], axis=1)
                s = s + dm @ cd
        elif self.kind == "video":
            active = 20 + 2 * (k // 5)
            a = g.standard_normal((active, b))
            s = np.einsum("mx,my,mc,mf->xycf", self.prof_x[:active], self.prof_y[:active], self.prof_c[:active], a,
                          optimize=True)
            s = np.reshape(np.asfortranarray(s), (-1, b), order="F")
        else:  # simulation
            s = self._simulation(k, b)
        s = _add_noise(g, s, self.noise)
        return np.asfortranarray(np.reshape(s, self.modes + (b,), order="F"))

    def _simulation(self, k: int, b: int) -> np.ndarray:
        t0 = k * b
        if self._ar_state is None or self._ar_t > t0:
            self._ar_rng = np.random.default_rng([self.seed, 2])
            nk = len(self.kvec)
            self._ar_state = self._ar_rng.standard_normal((3, nk)) + 1j * self._ar_rng.standard_normal((3, nk))
            self._ar_t = 0
        rho = 0.95
        sq = math.sqrt(1 - rho * rho)
        while self._ar_t < t0:
            self._advance_ar(rho, sq)
        g = self.grid
        out = np.empty((g ** 3 * 3, b))
        for j in range(b):
            F = np.zeros((3, g, g, g), dtype=np.complex128)
            for comp in range(3):
                F[comp][self.kidx] = self._ar_state[comp]
            u = np.real(np.fft.ifftn(F, axes=(1, 2, 3))) * (g ** 3)  # sum_k c_k e^{+2 pi i k.x/g}
            # u[c, x, y, z] -> first-index-fastest x, y, z, c
            out[:, j] = np.ravel(np.transpose(u, (1, 2, 3, 0)), order="F")
            self._advance_ar(rho, sq)
        return out

    def _advance_ar(self, rho: float, sq: float) -> None:
        nk = len(self.kvec)
        xi = self._ar_rng.standard_normal((3, nk)) + 1j * self._ar_rng.standard_normal((3, nk))
        self._ar_state = rho * self._ar_state + sq * xi
        self._ar_t += 1


class DeviceStream:
    """cfg3/cfg4 generator producing increments directly in HBM (torch, CUDA).

    Same construction as ``Stream`` (kind "drift_tt"); noise and coefficients
    come from a seeded torch CUDA generator, so the bytes differ from the
    host stream while the distribution is identical.  Returns flat contiguous
    float64 CUDA tensors in first-index-fastest order.
    """

    def __init__(self, seed: int = 0, modes: Sequence[int] = (8,) * 7, true_rank: int = 12, device: str = "cuda",
                 rank_shard: int = 0, drift_amp: float = 0.3, noise: float = 1e-3):
        import torch

        self.torch = torch
        self.host = Stream(3, seed=seed, modes=modes, true_rank=true_rank, drift_amp=drift_amp, noise=noise)
        self.modes = tuple(modes)
        self.device = device
        self.seed = seed
        self.rank_shard = rank_shard
        self.phi = torch.from_numpy(np.ascontiguousarray(self.host.phi.T)).to(device)  # r x S (row-major = S x r col-major)
        self._drifts = {}

    def _drift(self, j: int):
        if j not in self._drifts:
            self._drifts[j] = self.torch.from_numpy(self.host.drift(j)).to(self.device)
        return self._drifts[j]

    def increment(self, k: int, batch: int, out=None):
        """Flat (prod(modes) * batch) float64 CUDA tensor; observation slabs contiguous."""
        torch = self.torch
        S = int(np.prod(self.modes))
        gen = torch.Generator(device=self.device)
        gen.manual_seed(int(np.random.SeedSequence([self.seed, 1, k, self.rank_shard]).generate_state(1)[0]))
        r = self.phi.shape[0]
        c = torch.randn((batch, r), generator=gen, device=self.device, dtype=torch.float64)
        basis = self.phi
        ids = self.host.drift_ids(k)
        if ids:
            amp = self.host.drift_amp * math.sqrt(r)
            cd = amp * torch.randn((batch, len(ids)), generator=gen, device=self.device, dtype=torch.float64)
            c = torch.cat([c, cd], dim=1)
            basis = torch.cat([self.phi] + [self._drift(j)[None, :] for j in ids], dim=0)
        if out is None:
            out = torch.empty(S * batch, device=self.device, dtype=torch.float64)
        y = out.view(batch, S)
        torch.matmul(c, basis, out=y)  # row o = observation o (contiguous slab)
        sn = torch.linalg.vector_norm(y)
        nz = torch.randn((batch, S), generator=gen, device=self.device, dtype=torch.float64)
        nn = torch.linalg.vector_norm(nz)
        y.add_(nz, alpha=float(self.host.noise * sn / nn))
        del nz
        return out
