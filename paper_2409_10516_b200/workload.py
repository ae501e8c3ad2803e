"""GPU synthesis of the reference's OOD workload (workload.cpp:102-203).

Same algorithm and RNG streams as generate_workload: splitmix64 streams seeded
by mix_seed(seed, group+1, tag) (util.hpp:13-66), Box-Muller normals in pairs,
anisotropic hidden states, per-head query projections mixed by ood_strength
and the joint concentration scaling. splitmix64 is counter-based
(state_i = seed + i*golden), so each stream is generated in parallel on the
GPU. Differences to the CPU reference: device log/sin/cos/sqrt (<= 2 ulp) and
cuBLAS f64 GEMM summation order, so values agree to ~1e-15 relative before the
final f32 cast (tests/test_workload_gpu.py). Used for benchmark inputs at
scales where the CPU generator is too slow; parity tests use the oracle's
generator.
"""
from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np
import torch

GOLDEN = 0x9E3779B97F4A7C15
M64 = (1 << 64) - 1


def _to_i64(x: int) -> int:
    x &= M64
    return x - (1 << 64) if x >= 1 << 63 else x


def splitmix64_host(state: int) -> tuple[int, int]:
    state = (state + GOLDEN) & M64
    z = state
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & M64
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & M64
    return state, z ^ (z >> 31)


def mix_seed(seed: int, a: int, b: int = 0) -> int:
    s, h = splitmix64_host(seed)
    s = h ^ ((a * 0xD6E8FEB86659FD93) & M64)
    s, h = splitmix64_host(s)
    s = h ^ ((b * 0xCA5A826395121157) & M64)
    _, h = splitmix64_host(s)
    return h


def _lsr(x: torch.Tensor, k: int) -> torch.Tensor:
    return (x >> k) & ((1 << (64 - k)) - 1)


def splitmix_stream(seed: int, start: int, count: int, device) -> torch.Tensor:
    """Outputs start .. start+count-1 of the splitmix64 stream (int64 bits)."""
    i = torch.arange(start + 1, start + count + 1, dtype=torch.int64, device=device)
    z = i * _to_i64(GOLDEN) + _to_i64(seed)          # wraps mod 2^64
    z = (z ^ _lsr(z, 30)) * _to_i64(0xBF58476D1CE4E5B9)
    z = (z ^ _lsr(z, 27)) * _to_i64(0x94D049BB133111EB)
    return z ^ _lsr(z, 31)


def uniforms(bits: torch.Tensor) -> torch.Tensor:
    return _lsr(bits, 11).to(torch.float64) * (2.0 ** -53)


def normals(seed: int, count: int, device) -> torch.Tensor:
    """First `count` Rng::normal() draws of Rng(seed) (util.hpp:47-60)."""
    pairs = (count + 1) // 2
    u = uniforms(splitmix_stream(seed, 0, 2 * pairs, device)).view(pairs, 2)
    u1, u2 = u[:, 0], u[:, 1]
    # u1 == 0 (probability 2^-53 per pair) would shift the CPU stream by one draw
    r = torch.sqrt(-2.0 * torch.log(u1))
    th = (2.0 * math.pi) * u2
    out = torch.stack([r * torch.cos(th), r * torch.sin(th)], dim=1).reshape(-1)
    return out[:count]


class HostRng:
    """Sequential Rng for the few host-side draws (calibration indices)."""

    def __init__(self, seed: int):
        self.state = seed

    def uniform(self) -> float:
        self.state, z = splitmix64_host(self.state)
        return (z >> 11) * 2.0 ** -53

    def uniform_index(self, n: int) -> int:
        return int(self.uniform() * float(n)) % n


@dataclass
class WorkloadSpec:
    """types.hpp:37-50"""

    n_ctx: int = 8192
    d_model: int = 256
    d_head: int = 128
    n_heads: int = 1
    n_kv_groups: int = 1
    seed: int = 7
    ood_strength: float = 2.0
    concentration: float = 12.0
    n_decode: int = 256


def generate_group(spec: WorkloadSpec, g: int, device="cuda"):
    """One KV group: keys, values [n_ctx, d_head] and per-head prefill/decode
    queries [heads_per_group, n, d_head], all f32 on `device`."""
    hpg = spec.n_heads // spec.n_kv_groups
    DM, DH, N, ND = spec.d_model, spec.d_head, spec.n_ctx, spec.n_decode
    f64 = torch.float64

    def grng(tag):
        return mix_seed(spec.seed, g + 1, tag)

    scale = torch.sqrt(1.0 / torch.arange(1, DM + 1, dtype=f64, device=device))
    mu_dir = normals(grng(1), DM, device)
    mu_dir = mu_dir / torch.sqrt((mu_dir * mu_dir).sum())
    mu = (2.5 * math.sqrt(float((scale * scale).sum()))) * mu_dir
    h = mu + normals(grng(2), N * DM, device).view(N, DM) * scale
    hq = h + 0.25 * normals(grng(3), N * DM, device).view(N, DM) * scale
    hdec = mu + normals(grng(4), ND * DM, device).view(ND, DM) * scale
    hdec = hdec + 0.25 * normals(grng(5), ND * DM, device).view(ND, DM) * scale
    ps = 1.0 / math.sqrt(DM)
    s = spec.ood_strength
    mixn = 1.0 / math.sqrt(1.0 + s * s)
    w0 = normals(grng(6), DM * DH, device).view(DM, DH) * ps
    wk = (w0 + s * (normals(grng(7), DM * DH, device).view(DM, DH) * ps)) * mixn
    wv = normals(grng(8), DM * DH, device).view(DM, DH) * ps
    keys = h @ wk
    values = h @ wv
    del h
    qp, qd = [], []
    for m in range(hpg):
        head = g * hpg + m
        bq = normals(mix_seed(spec.seed, spec.n_kv_groups + head + 1, 100), DM * DH,
                     device).view(DM, DH) * ps
        wq = (w0 + s * bq) * mixn
        qp.append(hq @ wq)
        qd.append(hdec @ wq)
    c = 1.0
    if N > 0:
        cal = HostRng(grng(9))
        nqs, nks = min(256, N), min(8192, N)
        picks = [(cal.uniform_index(hpg), cal.uniform_index(N)) for _ in range(nqs)]
        kidx = [cal.uniform_index(N) for _ in range(nks)]
        qs = torch.stack([qp[m][r] for m, r in picks])
        ks = keys[torch.tensor(kidx, device=device)]
        z = (qs @ ks.T) / math.sqrt(DH)
        mean = z.mean(dim=1, keepdim=True)
        sig = torch.sqrt(((z - mean) ** 2).mean(dim=1)).mean().item()
        if sig > 0:
            c = math.sqrt(spec.concentration / sig)
    return dict(keys=(keys * c).float(), values=values.float(),
                prefill_q=torch.stack([(x * c).float() for x in qp]),
                decode_q=torch.stack([(x * c).float() for x in qd]))
