"""Synthetic clustered streams generated on the GPU (input source for benchmarks).

Same distributions as the reference generator (workload.cpp:56-187): unit keys
normalize(center + noise * N(0, I)) around per-(scene, domain) centers that mix the scene's
visual center (cross_modal_mix = 0.6), N(0, 1) values, unit queries near a center. Generated with
torch on the device (plumbing only); no parity requirement -- parity runs use the reference's own
generator through the oracle.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch


@dataclass
class ClusteredState:
    """A pre-clustered KV state for `ClusterKVCache.bulk_load`."""

    d: int
    L: int
    N: int
    C: int
    T: int
    keys: torch.Tensor       # [L, N, d] bf16/f32 on device
    values: torch.Tensor     # [L, N, d]
    assign: np.ndarray       # [L, N] int32 cluster index
    frame_ids: np.ndarray    # [N] int64
    token_ids: np.ndarray    # [N] int32
    centers: torch.Tensor    # [L, C, d] f32 unit
    visual: np.ndarray       # [d] f32 unit


def _unit(x: torch.Tensor) -> torch.Tensor:
    return x / x.norm(dim=-1, keepdim=True)


def clustered_state(L: int, N: int, C: int, d: int = 128, T: int = 196, noise: float = 0.015,
                    mix: float = 0.6, dtype=torch.bfloat16, seed: int = 42,
                    device: str = "cuda") -> ClusteredState:
    g = torch.Generator(device=device)
    g.manual_seed(seed)
    visual = _unit(torch.randn(d, generator=g, device=device))
    centers = _unit(mix * visual + (1 - mix) * _unit(torch.randn(L, C, d, generator=g, device=device)))
    n_frames = (N + T - 1) // T
    frame_of = torch.arange(N, device=device) // T
    # each frame's tokens sit near one cluster; clusters own contiguous runs of frames
    cl_of_frame = (torch.arange(n_frames, device=device) * C) // n_frames
    assign = cl_of_frame[frame_of]  # [N]
    keys = torch.empty(L, N, d, dtype=dtype, device=device)
    values = torch.empty(L, N, d, dtype=dtype, device=device)
    for l in range(L):
        k = centers[l, assign] + noise * torch.randn(N, d, generator=g, device=device)
        keys[l] = _unit(k).to(dtype)
        values[l] = torch.randn(N, d, generator=g, device=device).to(dtype)
    a = assign.to(torch.int32).cpu().numpy()
    return ClusteredState(d, L, N, C, T, keys, values, np.ascontiguousarray(np.broadcast_to(a, (L, N))),
                          (np.arange(N) // T).astype(np.int64), (np.arange(N) % T).astype(np.int32),
                          centers, visual.float().cpu().numpy())


def frames_near(state: ClusteredState, n_frames: int, first_frame: int, noise: float = 0.015,
                seed: int = 7, dtype=torch.bfloat16):
    """New frames [n, L, T, d]: each frame's tokens near one existing cluster of each domain."""
    dev = state.centers.device
    g = torch.Generator(device=dev)
    g.manual_seed(seed)
    L, T, d, C = state.L, state.T, state.d, state.C
    cl = torch.randint(0, C, (n_frames, L), generator=g, device=dev)
    base = state.centers[torch.arange(L, device=dev)[None, :], cl]  # [n, L, d]
    k = _unit(base[:, :, None, :] + noise * torch.randn(n_frames, L, T, d, generator=g, device=dev))
    v = torch.randn(n_frames, L, T, d, generator=g, device=dev)
    vis = torch.from_numpy(state.visual).to(dev)
    visual = _unit(vis[None, :] + 0.01 * torch.randn(n_frames, d, generator=g, device=dev))
    return (k.to(dtype).contiguous(), v.to(dtype).contiguous(), visual.float().cpu().numpy(),
            np.arange(first_frame, first_frame + n_frames, dtype=np.int64))


def queries_near(state: ClusteredState, n_steps: int, noise: float = 0.05, seed: int = 11):
    """Unit queries [n_steps, L, d] f32, each near a random cluster center of its domain."""
    dev = state.centers.device
    g = torch.Generator(device=dev)
    g.manual_seed(seed)
    L, d, C = state.L, state.d, state.C
    cl = torch.randint(0, C, (n_steps, L), generator=g, device=dev)
    base = state.centers[torch.arange(L, device=dev)[None, :], cl]
    return _unit(base + noise * torch.randn(n_steps, L, d, generator=g, device=dev)).float().contiguous()


def frames_drift(state: ClusteredState, n_frames: int, first_frame: int, noise: float = 0.02,
                 drift: float = 0.01, visual_noise: float = 0.05, seed: int = 17, dtype=torch.bfloat16):
    """New frames [n, L, T, d] with gen_stream's scene dynamics (workload.cpp:110-135): each
    domain's center starts at one existing cluster center and drifts by perturb(center, drift)
    every frame after the first; keys = normalize(center + noise * N(0, I)) (semantic_noise 0.02,
    drift_rate 0.01 as SURVEY §8(d) config 2 states), values N(0, 1), visual = perturb(visual
    center, visual_noise). At d = 128 a key's squared distance to its center is about noise^2 * d
    = 0.051 > tau_min = 0.05, so clusters of ~512 members are over the Eq. 5 threshold and the
    stream splits them: the maintenance regime, unlike `frames_near`'s absorb-only one."""
    dev = state.centers.device
    g = torch.Generator(device=dev)
    g.manual_seed(seed)
    L, T, d, C = state.L, state.T, state.d, state.C
    cl = torch.randint(0, C, (L,), generator=g, device=dev)
    center = state.centers[torch.arange(L, device=dev), cl].clone()  # [L, d]
    ks, vs = [], []
    vis = torch.from_numpy(state.visual).to(dev)
    visual = []
    for f in range(n_frames):
        if f > 0:
            center = _unit(center + drift * torch.randn(L, d, generator=g, device=dev))
        visual.append(_unit(vis + visual_noise * torch.randn(d, generator=g, device=dev)))
        ks.append(_unit(center[:, None, :] + noise * torch.randn(L, T, d, generator=g, device=dev)).to(dtype))
        vs.append(torch.randn(L, T, d, generator=g, device=dev).to(dtype))
    return (torch.stack(ks).contiguous(), torch.stack(vs).contiguous(),
            torch.stack(visual).float().cpu().numpy(),
            np.arange(first_frame, first_frame + n_frames, dtype=np.int64))
