"""Seeded synthetic inputs with the BASELINE.json config shapes and value
distributions (the paper's video / hyperspectral datasets are not available;
SURVEY.md §8d fixes the generators' free parameters, marked *proposal* there).

Host generators return Fortran-ordered numpy arrays (n1, n2, n3) and take any
shape, so tests can run the same distributions at oracle-sized scales. The
large device generators build the tensor directly in HBM with torch (data
synthesis is not part of the measured hot path).
"""
from __future__ import annotations

import math

import numpy as np

CONFIGS = {
    "cfg1": dict(n1=64, n2=48, n3=32, p=8, k=4),
    "cfg2": dict(n1=240, n2=320, n3=200, p=20, k=10, ks=(1, 5, 10, 20)),
    "cfg3": dict(n1=512, n2=512, n3=224, p=32, k=16),
    "cfg4": dict(n1=1024, m=512, n2=1024, n3=256, p=64),
    "cfg5": dict(n1=2048, n2=2048, n3=1024, p=128, k=32, rank=50, noise=1e-3),
}


def video(n1=240, n2=320, n3=200, seed=0, rank=10, blob_sigma=12.0, noise=0.01):
    """cfg2: smooth rank-10 background (outer products of sinusoids) + a
    unit Gaussian blob (sigma=12 px) moving on a linear path + N(0, 0.01^2)."""
    rng = np.random.default_rng(seed)
    i = np.arange(n1)[:, None]
    j = np.arange(n2)[None, :]
    bg = np.zeros((n1, n2))
    for _ in range(rank):
        a, b = rng.uniform(0.5, 3.0, 2)
        al = rng.uniform(0.5, 1.5)
        ph, ps = rng.uniform(0, 2 * math.pi, 2)
        bg += al * np.sin(2 * math.pi * a * i / n1 + ph) * np.sin(2 * math.pi * b * j / n2 + ps)
    x0, y0 = n1 / 6.0, n2 / 8.0
    x1, y1 = 5.0 * n1 / 6.0, 7.0 * n2 / 8.0
    out = np.empty((n1, n2, n3), order="F")
    for f in range(n3):
        t = f / max(1, n3 - 1)
        cx, cy = x0 + t * (x1 - x0), y0 + t * (y1 - y0)
        blob = np.exp(-((i - cx) ** 2 + (j - cy) ** 2) / (2 * blob_sigma ** 2))
        out[:, :, f] = bg + blob
    out += noise * rng.standard_normal(out.shape)
    return out


def hyperspectral(n1=512, n2=512, n3=224, seed=0, endmembers=6, noise_frac=0.01):
    """cfg3: per-pixel Dirichlet(1) mixture of 6 smooth endmember spectra
    (sums of 3 Gaussian bumps over the bands) + 1% Gaussian noise
    (sigma = 0.01 * RMS of the noiseless cube)."""
    rng = np.random.default_rng(seed)
    t = np.arange(n3)[None, :]
    E = np.zeros((endmembers, n3))
    for l in range(endmembers):
        for _ in range(3):
            h = rng.uniform(0.3, 1.0)
            c = rng.uniform(0, n3)
            s = rng.uniform(5.0, 25.0)
            E[l] += h * np.exp(-((t[0] - c) ** 2) / (2 * s * s))
    w = -np.log(rng.uniform(size=(n1 * n2, endmembers)))
    w /= w.sum(axis=1, keepdims=True)
    tubes = w @ E  # (N, n3), row i + j*n1 is the tube (i,j,:)
    rms = math.sqrt(float(np.mean(tubes ** 2)))
    tubes += noise_frac * rms * rng.standard_normal(tubes.shape)
    return np.asfortranarray(tubes.reshape(n1, n2, n3, order="F"))


def gaussian(n1, n2, n3, seed=0, stream=0):
    """cfg4 operands: i.i.d. N(0,1) (stream selects A=1 / B=2)."""
    rng = np.random.default_rng([seed, stream])
    return np.asfortranarray(rng.standard_normal((n1, n2, n3)))


def cp_tensor(n1=2048, n2=2048, n3=1024, rank=50, noise=1e-3, seed=0):
    """cfg5 (host, for scaled-down tests): rank-R CP tensor with N(0,1)
    factors + N(0, noise^2) (noise read as a standard deviation)."""
    rng = np.random.default_rng(seed)
    f1 = rng.standard_normal((n1, rank))
    f2 = rng.standard_normal((n2, rank))
    f3 = rng.standard_normal((n3, rank))
    kr = (f1[:, None, :] * f2[None, :, :]).reshape(n1 * n2, rank, order="F")
    tubes = kr @ f3.T
    tubes += noise * rng.standard_normal(tubes.shape)
    return np.asfortranarray(tubes.reshape(n1, n2, n3, order="F"))


# ------------------------------------------------------------ device (torch)
def _empty_f(shape, device):
    import torch
    rev = tuple(reversed(shape))
    return torch.empty(rev, dtype=torch.float64, device=device).permute(*reversed(range(len(shape))))


def gaussian_device(n1, n2, n3, seed=0, stream=0, device="cuda"):
    import torch
    g = torch.Generator(device=device)
    g.manual_seed(int(seed) * 1000003 + int(stream))
    flat = torch.empty(n1 * n2 * n3, dtype=torch.float64, device=device)
    flat.normal_(generator=g)
    return flat.view(n3, n2, n1).permute(2, 1, 0)


def cp_tensor_device(n1=2048, n2=2048, n3=1024, rank=50, noise=1e-3, seed=0, device="cuda",
                     out=None):
    """cfg5 on the device: tubes = KhatriRao(F1, F2) F3^T + noise, built
    slab by slab (no second full-size temporary)."""
    import torch
    g = torch.Generator(device=device)
    g.manual_seed(int(seed) * 7919 + 5)
    f1 = torch.randn(n1, rank, dtype=torch.float64, device=device, generator=g)
    f2 = torch.randn(n2, rank, dtype=torch.float64, device=device, generator=g)
    f3 = torch.randn(n3, rank, dtype=torch.float64, device=device, generator=g)
    kr = (f1[:, None, :] * f2[None, :, :]).permute(1, 0, 2).reshape(n1 * n2, rank)
    N = n1 * n2
    flat = out if out is not None else torch.empty(N * n3, dtype=torch.float64, device=device)
    tubes = flat.view(n3, N)  # row k = frontal slice k (column k of the tube matrix)
    step = max(1, (1 << 28) // N)
    for k0 in range(0, n3, step):
        k1 = min(n3, k0 + step)
        slab = tubes[k0:k1]
        torch.matmul(f3[k0:k1], kr.T, out=slab)
        if noise:
            slab.add_(torch.randn(slab.shape, dtype=torch.float64, device=device, generator=g),
                      alpha=noise)
    return flat.view(n3, n2, n1).permute(2, 1, 0)


def cp_block_device(n1, n2, n3, j0, nj, rank=50, noise=1e-3, seed=0, device="cuda"):
    """Lateral block A[:, j0:j0+nj, :] of the cfg5 CP tensor for one rank of a
    pixel-sharded run: the CP factors are common (same seed on every rank);
    the noise of the block is drawn from a (seed, j0) stream."""
    import torch
    g = torch.Generator(device=device)
    g.manual_seed(int(seed) * 7919 + 5)
    f1 = torch.randn(n1, rank, dtype=torch.float64, device=device, generator=g)
    f2 = torch.randn(n2, rank, dtype=torch.float64, device=device, generator=g)
    f3 = torch.randn(n3, rank, dtype=torch.float64, device=device, generator=g)
    f2 = f2[j0:j0 + nj]
    kr = (f1[:, None, :] * f2[None, :, :]).permute(1, 0, 2).reshape(n1 * nj, rank)
    Nb = n1 * nj
    flat = torch.empty(Nb * n3, dtype=torch.float64, device=device)
    tubes = flat.view(n3, Nb)
    gn = torch.Generator(device=device)
    gn.manual_seed(int(seed) * 1000003 + 17 + int(j0))
    step = max(1, (1 << 28) // Nb)
    for k0 in range(0, n3, step):
        k1 = min(n3, k0 + step)
        slab = tubes[k0:k1]
        torch.matmul(f3[k0:k1], kr.T, out=slab)
        if noise:
            slab.add_(torch.randn(slab.shape, dtype=torch.float64, device=device, generator=gn),
                      alpha=noise)
    return flat.view(n3, nj, n1).permute(2, 1, 0)


def cp_block(n1, n2, n3, j0, nj, rank=50, noise=1e-3, seed=0):
    """Host lateral block A[:, j0:j0+nj, :] of a cfg5-distributed tensor
    (rank-R CP with N(0,1) factors + N(0, noise^2)): the CPU baseline's
    pixel sample. Same distribution as cp_tensor_device, not the same bits."""
    rng = np.random.default_rng([seed, 5])
    f1 = rng.standard_normal((n1, rank))
    f2 = rng.standard_normal((n2, rank))[j0:j0 + nj]
    f3 = rng.standard_normal((n3, rank))
    kr = (f1[:, None, :] * f2[None, :, :]).reshape(n1 * nj, rank, order="F")
    T = kr @ f3.T
    T += noise * np.random.default_rng([seed, 17, j0]).standard_normal(T.shape)
    return np.asfortranarray(T.reshape(n1, nj, n3, order="F"))


def cp_slice(n1, n2, rank=50, noise=1e-3, seed=0, i=0):
    """Host n1 x n2 transform-domain slice of a cfg5-distributed tensor:
    A x3 q for a unit q is sum_r c_r f1_r f2_r^T + N(0, noise^2) with
    c_r = (F3^T q)_r ~ N(0, 1) (the CPU baseline's slice-SVD sample)."""
    rng = np.random.default_rng([seed, 29, i])
    f1 = rng.standard_normal((n1, rank))
    f2 = rng.standard_normal((n2, rank))
    c = rng.standard_normal(rank)
    return np.asfortranarray((f1 * c) @ f2.T + noise * rng.standard_normal((n1, n2)))
