"""Device-side generators for the BASELINE.json configs C1-C5 (synthetic, seeded).

These build the dense FP64 input directly in HBM with torch (the bench's
untimed setup), then compress it on the GPU.  Recipes follow BASELINE.json
``configs`` / SURVEY §8(d); the host oracle (oracle/configs.py) states the
same recipes in numpy for parity tests, where identical host tiles are fed
to both sides.  All five matrices are symmetric, so the row-major buffer is
also the column-major one the compression kernel reads.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch


@dataclass(frozen=True)
class Config:
    name: str
    family: str
    n: int
    b: int
    eps: float
    method: str
    seed: int = 0
    cap: int | None = None  # low-rank slab capacity (None: b)


CONFIGS = {
    "C1": Config("C1", "random16", 2048, 256, 1e-8, "mgs"),
    "C2": Config("C2", "laplace", 16384, 256, 1e-8, "blocked-hh"),
    "C3": Config("C3", "expcov", 32768, 512, 1e-8, "tiled-hh"),
    "C4": Config("C4", "invpoisson", 16384, 256, 1e-10, "tiled-hh"),
    "C5": Config("C5", "laplace", 65536, 1024, 1e-8, "tiled-hh", cap=256),  # ranks <= ~15
}


def _morton_order(x: np.ndarray, bits: int) -> np.ndarray:
    q = np.clip((x * (1 << bits)).astype(np.int64), 0, (1 << bits) - 1)
    key = np.zeros(len(x), dtype=np.int64)
    for t in range(bits):
        key |= ((q[:, 0] >> t) & 1) << (2 * t)
        key |= ((q[:, 1] >> t) & 1) << (2 * t + 1)
    return np.argsort(key, kind="stable")


def dense_device(cfg: Config, n: int | None = None, device="cuda") -> torch.Tensor:
    """n x n FP64 matrix of the config's family, resident on ``device``."""
    n = n or cfg.n
    dev = torch.device(device)
    if cfg.family == "laplace":
        d = torch.arange(n, device=dev, dtype=torch.float64)
        g = torch.zeros(n, dtype=torch.float64, device=dev)
        g[1:] = -torch.log(2.0 * torch.abs(torch.sin(np.pi * d[1:] / n))) / (2.0 * np.pi)
        g[0] = 1.0 + torch.sum(torch.abs(g[1:])) / n
        out = torch.empty((n, n), dtype=torch.float64, device=dev)
        idx = torch.arange(n, device=dev)
        rows = 4096
        for r0 in range(0, n, rows):
            r = idx[r0:r0 + rows, None]
            out[r0:r0 + rows] = g[(r - idx[None, :]) % n]
        return out
    if cfg.family == "expcov":
        x = np.random.default_rng(cfg.seed).uniform(0.0, 1.0, (n, 2))
        x = torch.from_numpy(np.ascontiguousarray(x[_morton_order(x, 21)])).to(dev)
        out = torch.empty((n, n), dtype=torch.float64, device=dev)
        rows = 2048
        for r0 in range(0, n, rows):
            a = x[r0:r0 + rows]
            dx = a[:, 0:1] - x[None, :, 0]
            dy = a[:, 1:2] - x[None, :, 1]
            out[r0:r0 + rows] = torch.exp(-torch.sqrt(dx * dx + dy * dy) / 0.1)
        out.diagonal().add_(1e-4)
        return out
    if cfg.family == "random16":
        from numpy.random import default_rng
        rng = default_rng(cfg.seed)
        b, p = cfg.b, n // cfg.b
        s = 10.0 ** (-np.arange(16) / 2.0)
        host = np.empty((n, n))
        for i in range(p):
            for j in range(p):
                if i == j:
                    t = rng.standard_normal((b, b))
                else:
                    u = np.linalg.qr(rng.standard_normal((b, 16)))[0]
                    v = np.linalg.qr(rng.standard_normal((b, 16)))[0]
                    t = (u * s) @ v.T
                host[i * b:(i + 1) * b, j * b:(j + 1) * b] = t
        return torch.from_numpy(host.T.copy()).to(dev)  # column-major storage
    if cfg.family == "invpoisson":
        g = int(round(np.sqrt(n)))
        h = 1.0 / (g + 1)
        k = np.arange(1, g + 1)
        s = np.sqrt(2.0 / (g + 1)) * np.sin(np.outer(k, k) * np.pi / (g + 1))
        lam = 2.0 - 2.0 * np.cos(k * np.pi / (g + 1))
        ix, iy = np.meshgrid(np.arange(g), np.arange(g), indexing="ij")
        ix, iy = ix.ravel(), iy.ravel()
        order = _morton_order(np.stack([ix, iy], 1).astype(float) / g, max(1, int(np.ceil(np.log2(g)))))
        ix, iy = ix[order], iy[order]
        S = torch.from_numpy(s).to(dev)
        w = (S[torch.from_numpy(ix).to(dev)][:, :, None] * S[torch.from_numpy(iy).to(dev)][:, None, :]).reshape(n, g * g)
        d = torch.from_numpy(((h * h) / (lam[:, None] + lam[None, :])).ravel()).to(dev)
        out = (w * d) @ w.T
        return 0.5 * (out + out.T)
    raise ValueError(cfg.family)
