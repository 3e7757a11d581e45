"""Full-size parity fixtures: the reference run over BASELINE configs at
their full sizes, stored per increment, and the checks the GPU tests apply.

A fixture (``tests/golden/<name>.npz``, written by
``tools/make_fullsize_fixtures.py`` with the reference library
oracle/_ref/libttref.so) holds, per increment k of the stream:

* ``sha256[k]``      SHA-256 of the increment's bytes (first-index-fastest);
* the reference's UpdateReport: ``ranks_after``, ``obs_used``, ``eps_target``,
  ``estimate``, ``clamped``;
* ``rre[k]``         the reference's metrics.cpp RRE of increment k under the
  train right after increment k (the increment's own reconstruction error);
* ``fp[k]``          subspace fingerprints f[i, j] = |Phi_iᵀ z_ij|² / |z_ij|²
  of every interface basis Phi_i (i = 1..d) on seeded probe vectors z_ij;
* ``recp[k]``        reconstruction probes zᵀ rec_o (N_PROBE x b) of increment
  k's observations under the train right after increment k, with
  ``recn[k]`` = |rec_o| and the probes' norms ``zn``;
* ``k{k}_core{i}``   the spatial cores after increment k (when small);

and the final train (``final_core{i}``, boundaries, ortho_count) when it is
small enough to commit.

A probe difference obeys |zᵀ(rec_g - rec_r)| <= |z| |rec_g - rec_r|, so
|dp| <= |z| |rec_o| 1e-10 is the probe form of "reconstruction within 1e-10"
(a failure proves a violation).

Tolerances follow tests/parity_util.py (1e-10).  A fingerprint moves to first
order by 2 sqrt(f) |dP| for a projector change |dP|, so |df| <= 2 sqrt(f) 1e-10
+ 1e-15 is the fingerprint form of "subspace distance <= 1e-10".
"""
from __future__ import annotations

import hashlib
import os
from typing import List, Sequence

import numpy as np

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
N_PROBE = 4
PROBE_SEED = 20260


def sha256_of(y) -> bytes:
    """SHA-256 of a host array's first-index-fastest bytes, or of a flat
    contiguous CUDA tensor (copied to host in chunks)."""
    h = hashlib.sha256()
    if isinstance(y, np.ndarray):
        h.update(np.asfortranarray(y).tobytes(order="F"))
        return h.digest()
    chunk = 1 << 27
    n = y.numel()
    for s in range(0, n, chunk):
        h.update(y[s:s + chunk].cpu().numpy().tobytes())
    return h.digest()


def left_unfoldings(cores: Sequence[np.ndarray]) -> List[np.ndarray]:
    return [np.reshape(c, (c.shape[0] * c.shape[1], c.shape[2]), order="F") for c in cores]


def fingerprints(cores: Sequence[np.ndarray], modes: Sequence[int]) -> np.ndarray:
    """f[i-1, j] = |Phi_iᵀ z|² / |z|² for interface i = 1..d (Phi_i is the
    n_1..n_i x r_i basis chained from cores 1..i), seeded probes z."""
    d = len(modes)
    us = left_unfoldings(cores[:d])
    out = np.zeros((d, N_PROBE))
    for k in range(1, d + 1):
        rows = int(np.prod(modes[:k]))
        z = np.random.default_rng([PROBE_SEED, k]).standard_normal((rows, N_PROBE))
        cur = np.reshape(z, (modes[0], -1), order="F")
        for i in range(k):
            nxt = us[i].T @ cur
            if i + 1 < k:
                cur = np.reshape(nxt, (us[i].shape[1] * modes[i + 1], -1), order="F")
        out[k - 1] = np.sum(nxt * nxt, axis=0) / np.sum(z * z, axis=0)
    return out


def _probe_vectors(rows: int) -> np.ndarray:
    return np.random.default_rng([PROBE_SEED, 999]).standard_normal((rows, N_PROBE))


def recon_probes(cores: Sequence[np.ndarray], modes: Sequence[int], lo: int, hi: int):
    """(zᵀ rec_o for o in [lo, hi), |rec_o|, |z|): rec_o = Phi c_o with the
    full spatial chain Phi (orthonormal, so |rec_o| = |c_o|)."""
    d = len(modes)
    us = left_unfoldings(cores[:d])
    z = _probe_vectors(int(np.prod(modes)))
    cur = np.reshape(z, (modes[0], -1), order="F")
    for i in range(d):
        nxt = us[i].T @ cur
        if i + 1 < d:
            cur = np.reshape(nxt, (us[i].shape[1] * modes[i + 1], -1), order="F")
    w = nxt  # Phiᵀ z: r_d x N_PROBE
    last = cores[d]
    c = np.reshape(last, (last.shape[0], -1), order="F")[:, lo:hi]
    return w.T @ c, np.linalg.norm(c, axis=0), np.linalg.norm(z, axis=0)


def recon_probes_agree(pg: np.ndarray, pr: np.ndarray, recn: np.ndarray, zn: np.ndarray,
                       tol: float = 1e-10) -> float:
    """Worst |dp| / (|z| |rec_o| tol + 1e-300) (<= 1 passes)."""
    bound = zn[:, None] * recn[None, :] * tol + 1e-300
    return float(np.max(np.abs(pg - pr) / bound))


def fingerprints_agree(fg: np.ndarray, fr: np.ndarray, tol: float = 1e-10) -> float:
    """Worst |df| / (2 sqrt(f) tol + 1e-15) (<= 1 passes)."""
    bound = 2.0 * np.sqrt(np.maximum(fg, fr)) * tol + 1e-15
    return float(np.max(np.abs(fg - fr) / bound))


def interface_gram(ca: Sequence[np.ndarray], cb: Sequence[np.ndarray]) -> np.ndarray:
    """Phi_aᵀ Phi_b for the full spatial chains (cores 1..d), contracted core by core."""
    m = np.ones((1, 1))
    for a, b in zip(ca, cb):
        # m_new[p, q] = sum_n sum_{s,t} a[s, n, p] m[s, t] b[t, n, q]
        t = np.einsum("st,tnq->snq", m, b)
        m = np.einsum("snp,snq->pq", a, t)
    return m


def coefficient_agreement(cores_g, cores_r, d: int, lo: int, hi: int) -> float:
    """|c_g - (Phi_gᵀ Phi_r) c_r| / |c_r| over observations [lo, hi): the part
    of |rec_g - rec_r| inside the GPU subspace (the rest is the subspace
    distance, checked separately)."""
    m = interface_gram(cores_g[:d], cores_r[:d])
    cg = np.reshape(cores_g[d], (cores_g[d].shape[0], -1), order="F")[:, lo:hi]
    cr = np.reshape(cores_r[d], (cores_r[d].shape[0], -1), order="F")[:, lo:hi]
    den = float(np.linalg.norm(cr))
    return float(np.linalg.norm(cg - m @ cr)) / (den if den > 0 else 1.0)


def load(name: str) -> dict:
    path = os.path.join(GOLD, name + ".npz")
    return dict(np.load(path, allow_pickle=False))


def final_cores(fx: dict) -> List[np.ndarray]:
    return [fx[f"final_core{i}"] for i in range(int(fx["n_cores"]))]


def step_cores(fx: dict, k: int) -> List[np.ndarray]:
    return [fx[f"k{k}_core{i}"] for i in range(int(fx["n_cores"]) - 1)]
