"""Checkpoint / resume of a training run ("torch.save of params, m, v, step and
RNG state"; the paper itself saves nothing but the 3DGS PLY).

A checkpoint holds theta (the packed 59-float-per-Gaussian parameters, R1), Adam's exp_avg
and exp_avg_sq, the step counter (Adam's bias corrections and the camera rotation depend on
it), the Gaussian count and SH degree, the host and device RNG states (the density step's
sampling draws from a torch generator), and an optional dict of caller data (e.g. the
per-camera scheduling hints, bgs_frame_save_hint).  Written to `path + ".tmp"` and renamed,
so a crash mid-write leaves the previous checkpoint intact.  load() checks the format and
every shape before returning, and raises ValueError on a truncated or inconsistent file.
Host-side plumbing only: no arithmetic of the method happens here.
"""
from __future__ import annotations

import os

import torch

FORMAT = 1
FLOATS_PER_GAUSSIAN = 59  # R1: mu 3, scale 3, rot 4, opacity 1, SH 48


def save(path: str, theta: torch.Tensor, exp_avg: torch.Tensor, exp_avg_sq: torch.Tensor, step: int, n: int,
         sh_degree: int, generators: dict[str, torch.Generator] | None = None, extra: dict | None = None) -> None:
    if theta.numel() != FLOATS_PER_GAUSSIAN * n or exp_avg.numel() != theta.numel() or \
            exp_avg_sq.numel() != theta.numel():
        raise ValueError("checkpoint.save: theta / exp_avg / exp_avg_sq must hold 59 n floats")
    state = {
        "format": FORMAT,
        "n": int(n),
        "sh_degree": int(sh_degree),
        "step": int(step),
        "theta": theta.detach().to("cpu", copy=True),
        "exp_avg": exp_avg.detach().to("cpu", copy=True),
        "exp_avg_sq": exp_avg_sq.detach().to("cpu", copy=True),
        "rng_host": torch.get_rng_state(),
        "rng_generators": {k: g.get_state() for k, g in (generators or {}).items()},
        "extra": {k: (v.detach().to("cpu", copy=True) if isinstance(v, torch.Tensor) else v)
                  for k, v in (extra or {}).items()},
    }
    tmp = f"{path}.tmp{os.getpid()}"
    torch.save(state, tmp)
    os.replace(tmp, path)


def load(path: str, device: torch.device | str = "cpu",
         generators: dict[str, torch.Generator] | None = None) -> dict:
    """The checkpoint's state with tensors on `device`; restores the host RNG and the states
    of the named generators passed in."""
    try:
        state = torch.load(path, map_location="cpu", weights_only=False)
    except Exception as e:  # noqa: BLE001 -- truncated / corrupt file
        raise ValueError(f"checkpoint.load: unreadable checkpoint {path}: {e}") from e
    if not isinstance(state, dict) or state.get("format") != FORMAT:
        raise ValueError(f"checkpoint.load: {path} is not a format-{FORMAT} checkpoint")
    n = state["n"]
    for k in ("theta", "exp_avg", "exp_avg_sq"):
        t = state[k]
        if not isinstance(t, torch.Tensor) or t.dtype != torch.float32 or t.numel() != FLOATS_PER_GAUSSIAN * n:
            raise ValueError(f"checkpoint.load: {k} of {path} does not hold 59 n = {59 * n} float32 values")
        state[k] = t.to(device).contiguous()
    if state["step"] < 0:
        raise ValueError("checkpoint.load: negative step")
    torch.set_rng_state(state["rng_host"])
    for k, g in (generators or {}).items():
        if k not in state["rng_generators"]:
            raise ValueError(f"checkpoint.load: no state for generator {k!r}")
        g.set_state(state["rng_generators"][k])
    state["extra"] = {k: (v.to(device) if isinstance(v, torch.Tensor) else v) for k, v in state["extra"].items()}
    return state
