#!/usr/bin/env python
"""bench.py -- BalanceGS hot path (3DGS differentiable tile rasterizer) on B200.

One step = one training iteration over a batch of B = 16 views of the garden-shaped
5.8M-Gaussian scene (BASELINE.json configs[3]/[4]): for each view preprocess -> sort ->
blend fwd -> L1 loss grad -> blend bwd -> preprocess bwd (grad +=), then (G > 1) an
NCCL all-reduce of grad[59N] and the fused Adam step.  The 16 views are split across
the G ranks (strong scaling: total work per step is fixed).  Every stage runs in
libbgs.so kernels through the C ABI; torch provides memory, streams and NCCL.

Prints ONE JSON line (rank 0).  `--impl reference` times the CPU oracle instead (the
reference arm of this tier) on a bounded sample of the same workload (one full view per step,
its per-pixel walks on a stratified 1/8 of the tiles).
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "fwd+bwd ms/view & views/s at 1/2/4/8 B200 (garden-shaped 5.8M Gaussians)"
UNIT = "views/s"
PEAKS_FALLBACK = {"hbm_gbs": 6650.0, "sm_max_mhz": 1965.0}
FP32_LANES_PER_SM = 128

# Algorithmic work per unit (DESIGN.md §6 restates each): FP32-pipe
# lane-ops per (pixel, list entry) pair of the per-pixel walk, by outcome
OPS_SKIPPED = 13        # power + exp + alpha test of an entry that is not blended
OPS_FWD_BLENDED = 20    # ... and the blend of one that is (forward)
OPS_BWD_BLENDED = 57    # backward: recompute, T division, colour / bg / geometric terms, 9 outputs


def _ncu_hw(config):
    """Hardware counters of the blend kernels from the committed ncu capture (garden camera 0,
    tools/profile_round.sh -> profiles/ncu_hw.json): FP32+ALU lane-ops executed and shared-memory
    wavefronts per launch, as fractions of the FP32-issue and shared-memory peaks at the SM
    clock ncu measured (148 SMs x 128 lanes; 1 wavefront per SM per clock)."""
    if config != "garden":
        return {}
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_hw.json")) as f:
            raw = json.load(f)
    except Exception:
        return {}
    out = {}
    for stage, d in raw.items():
        if not isinstance(d, dict) or not d.get("time_s"):
            continue
        clk = d["sm_hz"]
        e = {"hw_source": raw.get("_source", "profiles/ncu_hw.json")}
        if d.get("lane_ops"):
            e["hw_lane_op_frac"] = round(d["lane_ops"] / (d["time_s"] * 148 * FP32_LANES_PER_SM * clk), 4)
            e["hw_lane_ops_per_launch"] = d["lane_ops"]
        if d.get("smem_wavefronts"):
            e["smem_wavefront_frac"] = round(d["smem_wavefronts"] / (d["time_s"] * 148 * clk), 4)
        out[stage] = e
    return out


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=10)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--impl", default="ours", choices=["ours", "reference"])
    p.add_argument("--config", default="garden")
    p.add_argument("--views", type=int, default=16)
    p.add_argument("--num-gaussians", dest="n", type=int, default=None,
                   help="override the Gaussian count (debug only)")
    p.add_argument("--fuse-adam", action="store_true",
                   help="G = 1: the chain rule and Adam in one pass (bgs_preprocess_bwd_batch_adam; measured "
                        "slower at garden, 5.7 -> 8.3 ms per step, so off by default)")
    p.add_argument("--streams", type=int, default=2,
                   help="CUDA streams the step's views are spread over (round-robin; with the sorts and plans "
                        "ahead, measured at garden: 1 -> 331.8, 2 -> 345.5, 3 -> 345.4 views/s)")
    p.add_argument("--density-every", type=int, default=0,
                   help="run the NEXT-1 density-control step every D training steps (configs[4]; 0 = off)")
    p.add_argument("--update", default="sharded", choices=["sharded", "allreduce", "overlap"],
                   help="G > 1: reduce-scatter + Adam on a 1/G shard + all-gather (default); all-reduce + "
                        "full Adam on every rank; or 'overlap': the chain rule in Gaussian chunks, each chunk's "
                        "gradient all-reduced on a communication stream while the next computes (SURVEY 8(e) 1)")
    p.add_argument("--overlap-chunks", type=int, default=4, help="--update overlap: Gaussian chunks")
    p.add_argument("--sort-streams", type=int, default=8,
                   help="sort all of a step's views up front, round-robin over this many CUDA streams (their "
                        "latency-bound sort kernels overlap), then blend the views in order; 0 = each view's "
                        "sort inline before its forward (measured at garden: 0 -> 315.3, 2 -> 324.2, 4 -> 325.1, "
                        "8 -> 326.1 views/s; after the round-2 kernel work 4 -> 384.7, 8 -> 386.2; high stream "
                        "priority for the sorts: no change; waiting per view instead of for all sorts: no gain)")
    p.add_argument("--loss", default="l1dssim", choices=["l1dssim", "l1"],
                   help="per-view loss: the 3DGS 0.8 L1 + 0.2 D-SSIM (default) or L1 alone (R19)")
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--no-e2e", action="store_true")
    p.add_argument("--one-frame", action="store_true",
                   help="diagnostic: one frame for all views (no per-view scheduling hint)")
    p.add_argument("--serial-steps", type=int, default=3,
                   help="after the timed region, steps with every stage serialised on one stream, whose stage "
                        "times feed the per-stage rooflines (the timed region's stages overlap across streams)")
    p.add_argument("--no-consume", action="store_true",
                   help="keep the preprocess's zeroing of the blend-gradient slots instead of letting the chain "
                        "rule zero what it reads (bgs_frame_set_consume)")
    p.add_argument("--no-plan-ahead", action="store_true",
                   help="with --sort-streams: build each view's forward schedule in bgs_render_fwd and its "
                        "backward schedule in bgs_blend_bwd instead of ahead (with the sorts / beside the loss)")
    p.add_argument("--fixed-batch", action="store_true",
                   help="every step renders the same 16 cameras (views 4i mod 64), each frame hinted by its own "
                        "previous forward (round-1 bench); default: the batch rotates over the scene's cameras "
                        "(step s renders views 4i + s mod 64), each view hinted by its camera's last forward")
    p.add_argument("--sort-path", default="direct", choices=["direct", "radix_split", "rowsplit", "onesweep64"],
                   help="a4-a6 implementation (default: the direct tile split; the others are bit-identical)")
    p.add_argument("--seg-len", type=int, default=0,
                   help="blend work-unit segment length (bgs_frame_set_seg_len); 0 = the library's default")
    p.add_argument("--hints", default="camera", choices=["none", "camera"],
                   help="forward scheduling hint of the rotating batch: the camera's last forward "
                        "(bgs_frame_save_hint / load_hint: heavy-first order and speculative splits of walks "
                        "longer than 4 segments) or none (work ordered by the tile list lengths, no splits: "
                        "as fast in the overlapped step, 394.9 vs 393.5 views/s, but each forward alone "
                        "0.87 instead of 0.68 ms at garden)")
    p.add_argument("--no-assign", action="store_true",
                   help="A/B: accumulate the chain rule into a zeroed grad and zero it in Adam (the round-2 "
                        "default before bgs_preprocess_bwd_batch_assign)")
    p.add_argument("--no-variants", action="store_true",
                   help="skip the extra timed loops (fixed batch; rotating batch without scheduling hints)")
    p.add_argument("--pre-per-view", action="store_true",
                   help="diagnostic: one preprocess launch per view instead of one per 16 views")
    p.add_argument("--no-stage-events", action="store_true", help="diagnostic: no per-stage events in the timed loop")
    return p.parse_args()


def nccl_summary():
    """The lines of this process's NCCL log (NCCL_DEBUG_FILE) that identify the communicator:
    ranks, NVLS (in-switch reduction) support, channels / rings."""
    import glob

    path = os.environ.get("NCCL_DEBUG_FILE", "")
    files = glob.glob(path.replace("%h", "*").replace("%p", str(os.getpid()))) if path else []
    keep = []
    for fn in files[:1]:
        try:
            for ln in open(fn, errors="replace"):
                if any(k in ln for k in ("NVLS", "nRanks", "Init COMPLETE", "NCCL version", "Channel 00", "Trees",
                                          "P2P/CUMEM", "via P2P", "NVLink")):
                    keep.append(ln.strip()[-200:])
                if len(keep) >= 24:
                    break
        except OSError:
            pass
    return {"log": files[:1], "lines": keep}


def load_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return json.load(f), "measured"
    except Exception:
        return PEAKS_FALLBACK, "fallback"


def _update_desc(args, world):
    if world > 1:
        return {"sharded": "reduce-scatter + sharded Adam + all-gather", "allreduce": "all-reduce + Adam",
                "overlap": f"chain rule in {args.overlap_chunks} Gaussian chunks, each chunk's all-reduce overlapped "
                           "with the next, + Adam"}[args.update]
    if args.fuse_adam and not args.one_frame and args.views <= 16:
        return "chain rule fused with Adam"
    return "all-reduce (none at G = 1) + Adam"


def arm_config(scene, args, world):
    """The workload description shared by both arms (ours and --impl reference)."""
    cam = scene.cameras[0]
    return {"workload": f"{scene.name}-shaped {scene.n} Gaussians, {cam.width}x{cam.height}, SH degree "
                        f"{scene.sh_degree}, batch of {args.views} views per step (fwd+bwd each, then "
                        f"{_update_desc(args, world)})",
            "views_per_step": args.views, "n_gaussians": scene.n, "width": cam.width, "height": cam.height,
            "parallelism": f"view-dp{world}", "l2": f"inputs larger than L2 (theta {236 * scene.n / 1e9:.2f} GB, L2 126 MB)",
            "loss": "0.8 L1 + 0.2 D-SSIM (11x11 Gaussian window)" if args.loss == "l1dssim" else "L1",
            "density_every": args.density_every}


def _device_index(local_rank):
    """cuda device of this rank; BGS_FORCE_DEVICE pins every rank to one GPU (test-only)."""
    forced = os.environ.get("BGS_FORCE_DEVICE")
    return int(forced) if forced is not None else local_rank


def batch_views(n_views, n_cams, step=0):
    """views 4i + step mod n_cams for i < n_views (SURVEY §8(d) at step 0; the batch rotates
    with the step so that a 16-view batch visits each of 64 cameras every 4 steps)."""
    return [(4 * i + step) % n_cams for i in range(n_views)]


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    FIELDS = ["clocks.sm", "clocks.max.sm", "clocks_event_reasons.hw_slowdown",
              "clocks_event_reasons.hw_thermal_slowdown", "clocks_event_reasons.sw_thermal_slowdown",
              "clocks_event_reasons.sw_power_cap"]

    def __init__(self, index):
        self.index = index
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", f"--id={self.index}", "--query-gpu=" + ",".join(self.FIELDS),
                                          "--format=csv,noheader,nounits", "-lms",
                                          os.environ.get("BGS_CLOCK_SAMPLE_MS", "250")],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [x.strip() for x in ln.split(",")]
            if len(parts) != 6:
                continue
            try:
                sm.append(float(parts[0]))
                mx.append(float(parts[1]))
            except ValueError:
                continue
            for nm, val in zip(names, parts[2:]):
                if val.lower().startswith("active"):
                    reasons.add(nm)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"], "samples": 0}
        return {"sm_mhz": float(np.median(sm)), "sm_max_mhz": float(max(mx)), "reasons": sorted(reasons),
                "samples": len(sm)}


# ---------------------------------------------------------------------------- ours
def run_ours(args, rank, world, local_rank):
    import torch
    import torch.distributed as dist

    import gen
    import paper_2510_14564_b200 as bgs
    from paper_2510_14564_b200 import dp

    dev = torch.device("cuda", _device_index(local_rank))
    torch.cuda.set_device(dev)
    kw = {} if args.n is None else {"n": args.n}
    scene = gen.make(args.config, **kw)
    n = scene.n
    cams_all = scene.cameras
    n_cams = len(cams_all)

    def rank_cams(step, fixed=None):
        """camera indices of this rank's views at training step `step` (1-based)"""
        fixed = args.fixed_batch if fixed is None else fixed
        return dp.views_for_rank(batch_views(args.views, n_cams, 0 if fixed else step - 1), rank, world)

    n_mine = len(rank_cams(1))
    used = sorted(set(rank_cams(1, True)) if args.fixed_batch else range(n_cams))  # cameras any step renders
    W, H = cams_all[0].width, cams_all[0].height
    sharded = world > 1 and args.update == "sharded"
    overlap = world > 1 and args.update == "overlap" and not args.one_frame
    comm_stream = torch.cuda.Stream(device=dev) if overlap else None
    chunk_ev = [torch.cuda.Event() for _ in range(max(1, args.overlap_chunks))]
    # one GPU, one chain-rule launch: a10 and a11 fused (no collective between them)
    fused = world == 1 and not args.one_frame and args.fuse_adam and args.views <= 16
    # the step's single batched chain rule assigns grad, so grad is never read by it nor
    # zeroed by Adam (bgs_preprocess_bwd_batch_assign / bgs_adam_step_keep_grad)
    assign = not (args.one_frame or overlap or fused or args.no_assign)
    # the step's views share theta: one preprocess pass over it for all of them
    batch_pre = not args.one_frame and not args.pre_per_view
    total = 59 * n
    if sharded:
        # reduce-scatter -> Adam on this rank's 1/G shard -> all-gather: theta
        # and grad padded to G equal 16-byte-aligned shards; Adam moments for the shard only
        shard, padded = dp.shard_layout(total, world)
        sh_lo, sh_hi = dp.shard_range(rank, world, total)
        theta = torch.zeros(padded, dtype=torch.float32, device=dev)
        theta[:total].copy_(torch.from_numpy(scene.theta))
        m = torch.zeros(shard, dtype=torch.float32, device=dev)
    else:
        theta = torch.from_numpy(scene.theta).to(dev)
        m = torch.zeros_like(theta)
    dp.broadcast_params(theta, world)  # replicas start identical
    grad = torch.zeros_like(theta)
    v = torch.zeros_like(m)
    hp = bgs.AdamHParams(lr_means=1.6e-4 * scene.extent)
    deg = scene.sh_degree

    # size the key capacity once over every camera a step may render (overflow -> re-run
    # with a larger workspace, R25); each camera's scheduling hint (its forward's per-block
    # walk costs) is saved as a trainer keeps it, so every view is hinted by its camera's
    # last forward (bgs_frame_save_hint / bgs_frame_load_hint)
    dflags = {"direct": 0, "radix_split": bgs.BGS_DEBUG_SORT_RADIX_SPLIT, "rowsplit": bgs.BGS_DEBUG_SORT_ROWSPLIT,
              "onesweep64": bgs.BGS_DEBUG_SORT_ONESWEEP64}[args.sort_path]
    rend = bgs.Renderer(n, W, H, max_keys=1 << 24, device=dev, debug_flags=dflags)
    kmax = 0
    for c in used:
        rend.forward(theta, cams_all[c], deg)
        kmax = max(kmax, rend.num_keys)
    if int(kmax * 1.1) + 4096 > rend.max_keys:
        rend.alloc(int(kmax * 1.1) + 4096)
    hint_bytes = bgs.bgs_frame_hint_bytes(rend.frame)
    hints = {}
    for c in used:
        rend.forward(theta, cams_all[c], deg, check=False)
        hints[c] = torch.empty(hint_bytes, dtype=torch.uint8, device=dev)
        bgs.bgs_frame_save_hint(rend.frame, hints[c])
    # one frame per view slot of the batch
    rends = [rend] + [rend if args.one_frame else bgs.Renderer(n, W, H, max_keys=rend.max_keys, device=dev, debug_flags=dflags)
                      for _ in range(n_mine - 1)]

    # targets: a perturbed copy of theta rendered once, 8-bit (R19)
    r = gen.rng(1234)
    th_t = scene.theta.copy()
    seg = gen.segments(th_t, n)
    seg["sh"][:, 0, :] += 0.05 * r.standard_normal((n, 3)).astype(np.float32)
    seg["means"][:] += (0.01 * scene.extent * r.standard_normal((n, 3))).astype(np.float32)
    th_t_dev = torch.from_numpy(th_t).to(dev)
    targets = {}
    for c in used:
        out = rend.forward(th_t_dev, cams_all[c], deg)
        targets[c] = (out["image"].clamp(0, 1) * 255 + 0.5).to(torch.uint8).contiguous()
    del th_t_dev
    targets_host = {c: t.cpu().pin_memory() for c, t in targets.items()}
    targets_e2e = [torch.empty_like(targets[used[0]]) for _ in range(n_mine)]
    dl = torch.empty((3, H, W), dtype=torch.float32, device=dev)
    loss = torch.zeros(1, dtype=torch.float32, device=dev)
    loss_host = torch.zeros(1, dtype=torch.float32).pin_memory()
    scale = 1.0 / (3.0 * W * H * args.views)
    loss_ws = (torch.empty(bgs.bgs_loss_workspace_bytes(W, H), dtype=torch.uint8, device=dev)
               if args.loss == "l1dssim" else None)
    cam_structs_all = {c: bgs.camera(cams_all[c]) for c in used}
    stream = torch.cuda.current_stream()
    # views run round-robin on S streams (their frames, dL/dimage and loss workspaces are
    # independent): one view's single-CTA planning kernels and kernel tails overlap another
    # view's work; the batch's chain rule and update wait for all of them
    n_streams = 1 if args.one_frame else max(1, args.streams)
    side = [torch.cuda.Stream(device=dev) for _ in range(n_streams - 1)]
    streams_all = [stream] + side
    dls = [dl] + [torch.empty_like(dl) for _ in side]
    loss_wss = [loss_ws] + [None if loss_ws is None else torch.empty_like(loss_ws) for _ in side]
    fork_ev = torch.cuda.Event()
    join_evs = [torch.cuda.Event() for _ in side]
    sort_ahead = args.sort_streams > 0 and not args.one_frame
    sort_streams = [torch.cuda.Stream(device=dev) for _ in range(args.sort_streams)] if sort_ahead else []
    sort_evs = [torch.cuda.Event() for _ in range(n_mine)] if sort_ahead else []
    # the blend kernels' schedules built off the critical path: the forward's with the sorts,
    # the backward's on a side stream while the view's loss runs
    plan_ahead = sort_ahead and not args.no_plan_ahead
    plan_stream = torch.cuda.Stream(device=dev) if plan_ahead else None
    fwd_evs = [torch.cuda.Event() for _ in range(n_mine)] if plan_ahead else []
    plan_evs = [torch.cuda.Event() for _ in range(n_mine)] if plan_ahead else []
    stage_names = ["preprocess", "sort", "render_fwd", "loss", "blend_bwd", "preprocess_bwd", "allreduce", "adam"]
    if args.density_every:
        stage_names.append("density")
    # all timing events of the timed region are created up front (creating them inside the
    # loop adds host work between launches)
    n_marks = args.steps * (7 * n_mine + 11)
    pool = [torch.cuda.Event(enable_timing=True) for _ in range(n_marks)]
    step_no = [0]

    # the training state; the periodic density-control step (NEXT-1, --density-every)
    # replaces it with one of another size
    S = {"theta": theta, "grad": grad, "m": m, "v": v, "n": n, "rends": rends,
         "lo": sh_lo if sharded else 0, "hi": sh_hi if sharded else 59 * n}

    def derive():
        S["gs"] = bgs.gaussians(S["theta"][:59 * S["n"]], S["n"], deg)  # (sharded: theta is padded)
        S["frames"] = [rj.frame for rj in S["rends"]]
        if not args.one_frame and not args.no_consume:  # the batched chain rule zeroes what it reads
            for f in S["frames"]:
                bgs.bgs_frame_set_consume(f, True)
        if args.seg_len:
            for f in S["frames"]:
                bgs.bgs_frame_set_seg_len(f, args.seg_len)

    derive()
    del theta, grad, m, v, rends
    dens_prm = None
    dens_log = []
    if args.density_every:
        # r = the median 8-NN distance of the initial scene, estimated from a
        # 100k-point sample (8-NN distances scale as (sample / n)^(1/3) under thinning)
        from scipy.spatial import cKDTree

        mu = gen.segments(scene.theta, n)["means"]
        sub = mu[gen.rng(77).choice(n, min(n, 100_000), replace=False)].astype(np.float64)
        d8 = cKDTree(sub).query(sub, k=9)[0][:, 8]
        dens_prm = bgs.DensityParams(float(np.median(d8) * (len(sub) / n) ** (1.0 / 3.0)))

    def rebuild(theta_full, m_full, v_full, n_new, max_keys):
        # theta / Adam moments of n_new Gaussians (unpadded 59 n_new) into the layout of this
        # run (sharded: padded theta and grad, moments of this rank's shard), new frames
        tot = 59 * n_new
        old = S.pop("rends")
        S.pop("frames", None)
        del old
        if sharded:
            shard, padded = dp.shard_layout(tot, world)
            lo, hi = dp.shard_range(rank, world, tot)
            th = torch.zeros(padded, dtype=torch.float32, device=dev)
            th[:tot].copy_(theta_full)
            mm = torch.zeros(padded, dtype=torch.float32, device=dev)
            vv = torch.zeros(padded, dtype=torch.float32, device=dev)
            mm[:tot].copy_(m_full)
            vv[:tot].copy_(v_full)
            S["m"], S["v"] = mm[lo:hi].clone(), vv[lo:hi].clone()
            S["lo"], S["hi"] = lo, hi
        else:
            th = theta_full.clone()
            S["m"], S["v"] = m_full.clone(), v_full.clone()
            S["lo"], S["hi"] = 0, tot
        S["theta"], S["grad"], S["n"] = th, torch.zeros_like(th), n_new
        r0 = bgs.Renderer(n_new, W, H, max_keys=max_keys, device=dev, debug_flags=dflags)
        S["rends"] = [r0] + [r0 if args.one_frame else bgs.Renderer(n_new, W, H, max_keys=max_keys, device=dev, debug_flags=dflags)
                             for _ in range(n_mine - 1)]
        for c in hints:  # a new scene: no camera has a hint for it yet
            hint_ok[c] = False
        derive()

    def full_moments():
        tot = 59 * S["n"]
        if not sharded:
            return S["m"][:tot], S["v"][:tot]
        shard, padded = dp.shard_layout(tot, world)
        mf = torch.empty(padded, dtype=torch.float32, device=dev)
        vf = torch.empty(padded, dtype=torch.float32, device=dev)
        dist.all_gather_into_tensor(mf, S["m"])
        dist.all_gather_into_tensor(vf, S["v"])
        return mf[:tot], vf[:tot]

    def density_step():
        # NEXT-1 (§III-C): the same deterministic step on every rank (identical
        # theta and moments, the variates from a generator seeded by the step number)
        n0 = S["n"]
        mf, vf = full_moments()
        g = torch.Generator(device=dev)
        g.manual_seed(1000 + step_no[0])
        th2, m2, v2, n2, rep, _, _ = bgs.density_control(S["theta"][:59 * n0], mf, vf, n0, dens_prm, g)
        mk = int(S["rends"][0].max_keys * max(1.0, n2 / n0)) + 4096
        rebuild(th2, m2, v2, n2, mk)
        dens_log.append({"step": step_no[0], "n_before": n0, "n_after": n2, "pairs": int(rep.n_pairs),
                         "children": int(rep.n_children)})

    hint_ok = {c: True for c in hints}

    def one_step(tgts, record=None, tgt_events=None, hint_mode="camera", serial=False):
        """one training step; tgts(j, c) -> the target of view slot j (camera c).  hint_mode:
        "camera" (each view hinted by its camera's last forward), "slot" (by its frame's
        previous forward), "none" (no hint: work ordered by list length).  serial: every
        stage of every view in order on one stream (the per-stage timing pass)"""
        n_st = 1 if serial else n_streams
        side_ = [] if serial else side
        s_ahead = sort_ahead and not serial
        p_ahead = plan_ahead and not serial
        step_no[0] += 1
        cams_idx = rank_cams(step_no[0])
        cam_structs = [cam_structs_all[c] for c in cams_idx]

        def mark(marks):
            if record is not None:
                e = record["pool"][record["next"]]
                record["next"] += 1
                e.record()  # on the current stream (the view's)
                marks.append(e)

        gs, grad, frames = S["gs"], S["grad"], S["frames"]
        if batch_pre:  # a1-a3 for all of the step's views in one pass over theta
            marks = []
            mark(marks)
            bgs.bgs_preprocess_batch(gs, cam_structs, frames)
            mark(marks)
            if record is not None:
                record["marks"].append(("pre", marks))
        if s_ahead:  # a4-a6 of every view first, spread over the sort streams
            marks = []
            mark(marks)
            if p_ahead and hint_mode != "slot":  # the hints first: the plans follow them
                for j, c in enumerate(cams_idx):
                    bgs.bgs_frame_load_hint(frames[j], hints[c] if hint_mode == "camera" and hint_ok[c] else None)
            fork_ev.record(stream)
            for ss in sort_streams:
                ss.wait_event(fork_ev)
            for j in range(len(cam_structs)):
                with torch.cuda.stream(sort_streams[j % len(sort_streams)]):
                    bgs.bgs_sort(frames[j])
                    if p_ahead:
                        bgs.bgs_render_fwd_plan(frames[j])
                    sort_evs[j].record()
            for ev in sort_evs[:len(cam_structs)]:
                stream.wait_event(ev)
            mark(marks)
            if record is not None:
                record["marks"].append(("sort", marks))
        if side_:
            fork_ev.record(stream)
            for sj in side_:
                sj.wait_event(fork_ev)
        for j, cs in enumerate(cam_structs):
            rj = S["rends"][j]
            sj = streams_all[j % n_st]
            dl, loss_ws = dls[j % n_st], loss_wss[j % n_st]
            with torch.cuda.stream(sj):
                marks = []
                mark(marks)
                if not batch_pre:
                    bgs.bgs_preprocess(gs, cs, rj.frame)
                mark(marks)
                if not s_ahead:
                    bgs.bgs_sort(rj.frame)
                mark(marks)
                c = cams_idx[j]
                if p_ahead:
                    pass  # loaded before the sorts
                elif hint_mode == "camera":
                    bgs.bgs_frame_load_hint(rj.frame, hints[c] if hint_ok[c] else None)
                elif hint_mode == "none":
                    bgs.bgs_frame_load_hint(rj.frame, None)
                bgs.bgs_render_fwd(rj.frame, rj.image, rj.final_T, rj.n_contrib)
                if p_ahead:  # the backward's schedule, beside the loss
                    fwd_evs[j].record(sj)
                    plan_stream.wait_event(fwd_evs[j])
                    with torch.cuda.stream(plan_stream):
                        bgs.bgs_blend_bwd_plan(rj.frame)
                        plan_evs[j].record()
                if hint_mode == "camera":
                    bgs.bgs_frame_save_hint(rj.frame, hints[c])
                    hint_ok[c] = True
                mark(marks)
                if tgt_events is not None:  # this view's target has arrived (H2D on the copy stream)
                    sj.wait_event(tgt_events[j])
                tg = tgts(j, c)
                if loss_ws is not None:  # the 3DGS loss 0.8 L1 + 0.2 D-SSIM (NEXT-2), batch mean
                    bgs.bgs_l1_dssim_loss_grad(rj.image, tg, W, H, 0.2, 1.0 / args.views, dl, loss, loss_ws)
                else:  # L1 (R19)
                    bgs.bgs_l1_loss_grad(rj.image, tg, W, H, scale, dl, loss)
                mark(marks)
                if p_ahead:
                    sj.wait_event(plan_evs[j])
                bgs.bgs_blend_bwd(rj.frame, dl, rj.final_T, rj.n_contrib)
                mark(marks)
                if args.one_frame:  # the frame is reused by the next view: chain rule now
                    bgs.bgs_preprocess_bwd(gs, rj.frame, grad)
                mark(marks)
                if record is not None:
                    record["marks"].append(("view", marks))
        for sj, ev in zip(side_, join_evs):
            ev.record(sj)
            stream.wait_event(ev)
        marks = []
        mark(marks)
        theta, m, v, n, lo, hi = S["theta"], S["m"], S["v"], S["n"], S["lo"], S["hi"]
        if fused:  # a10 + a11 in one pass per Gaussian: the gradient never reaches memory
            bgs.bgs_preprocess_bwd_batch_adam(gs, frames, theta, None, m, v, hp, step_no[0])
        elif overlap:  # a10 in Gaussian chunks; chunk k's all-reduce runs while chunk k+1 computes
            for ci, (b, e) in enumerate(dp.gaussian_chunks(n, args.overlap_chunks)):
                bgs.bgs_preprocess_bwd_batch_range(gs, frames, grad, b, e - b)
                chunk_ev[ci].record(stream)
                comm_stream.wait_event(chunk_ev[ci])
                with torch.cuda.stream(comm_stream):
                    dp.allreduce_chunk(grad, n, b, e, world)
        elif not args.one_frame:  # a10 once over the batch's views: theta/grad cross HBM once
            if assign:  # grad = the batch's sum: never read, never zeroed
                bgs.bgs_preprocess_bwd_batch_assign(gs, frames, grad)
            else:
                bgs.bgs_preprocess_bwd_batch(gs, frames, grad)
        mark(marks)
        if fused:
            mark(marks)
            mark(marks)
        elif overlap:
            stream.wait_stream(comm_stream)  # the last chunk's exchange
            mark(marks)
            bgs.bgs_adam_step(theta, grad, m, v, n, hp, step_no[0])
            mark(marks)
        elif sharded:  # NCCL over NVLink: reduce-scatter, Adam on the shard, all-gather
            g_shard = dp.reduce_scatter_grads(grad, rank, world)
            mark(marks)
            bgs.bgs_adam_step_range(theta[lo:hi], g_shard, m, v, n, lo, hi - lo, hp, step_no[0])
            if not assign:
                bgs.bgs_zero(grad)  # the rest of grad still holds this rank's partial sums
            mark(marks)
            dp.all_gather_params(theta, rank, world)
        else:
            dp.allreduce_grads(grad, world)  # NCCL over NVLink (one exchange per batch)
            mark(marks)
            if assign:
                bgs.bgs_adam_step_keep_grad(theta, grad, m, v, n, hp, step_no[0])
            else:
                bgs.bgs_adam_step(theta, grad, m, v, n, hp, step_no[0])
            mark(marks)
        mark(marks)
        if args.density_every and step_no[0] % args.density_every == 0:
            density_step()  # periodic (configs[4]); changes n
        mark(marks)
        if record is not None:
            record["marks"].append(("batch", marks))

    def barrier():
        if world > 1:
            dist.barrier()

    dev_targets = lambda j, c: targets[c]  # noqa: E731  (device-resident inputs)

    # warm-up
    for _ in range(args.warmup):
        one_step(dev_targets)
    torch.cuda.synchronize()

    # the step trains theta (Adam), which changes the workload; the e2e loop and the variants
    # restart from this snapshot so every loop times the same sequence of training states
    mf, vf = full_moments()
    snap = (S["theta"][:59 * S["n"]].clone(), mf.clone(), vf.clone(), S["n"], step_no[0], S["rends"][0].max_keys)
    del mf, vf
    hints_snap = {c: (h.clone(), hint_ok[c]) for c, h in hints.items()}

    def restore():
        rebuild(snap[0], snap[1], snap[2], snap[3], snap[5])
        step_no[0] = snap[4]
        for c, (h, ok) in hints_snap.items():
            hints[c].copy_(h)
            hint_ok[c] = ok
        torch.cuda.synchronize()

    def check_overflow(what):
        for rj in S["rends"]:  # the sticky flag covers every step since the last check
            st, _ = bgs.bgs_frame_status(rj.frame)
            assert st == bgs.BGS_OK, f"key capacity overflow in the {what}"

    def max_over_ranks(ms):
        if world > 1:
            t = torch.tensor([ms], device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            ms = float(t.item())
        return ms

    check_overflow("warm-up")
    # the stage times come from a serial pass after the timed region when the step overlaps
    # views on streams; the timed region then records no stage events (their host calls
    # would slow small configs' launch-bound steps)
    concurrent = n_streams > 1 or sort_ahead
    serial_pass = concurrent and args.serial_steps > 0 and not args.no_stage_events and not args.density_every
    # ---- device-resident timed region (inputs larger than L2: theta 1.37 GB, keys GBs)
    record = {"next": 0, "marks": [], "pool": pool}
    barrier()
    torch.cuda.synchronize()
    launches0 = bgs.launch_count()
    t0 = torch.cuda.Event(enable_timing=True)
    t1 = torch.cuda.Event(enable_timing=True)
    hint_mode = "slot" if args.fixed_batch else args.hints
    with ClockSampler(_device_index(local_rank)) as clk:
        torch.cuda.nvtx.range_push("bench_timed")  # ncu --nvtx --nvtx-include "bench_timed/"
        t0.record(stream)
        for _ in range(args.steps):
            one_step(dev_targets, None if (args.no_stage_events or serial_pass) else record, hint_mode=hint_mode)
        t1.record(stream)
        torch.cuda.nvtx.range_pop()
        torch.cuda.synchronize()
    barrier()
    launches = bgs.launch_count() - launches0
    ms_local = t0.elapsed_time(t1)
    check_overflow("timed region")
    def stage_means(rec, steps):
        sums = {s: 0.0 for s in stage_names}
        for kind, mk in rec["marks"]:
            if kind == "pre":
                sums["preprocess"] += mk[0].elapsed_time(mk[1])
            elif kind == "sort":
                sums["sort"] += mk[0].elapsed_time(mk[1])
            elif kind == "view":
                for s, a, b in zip(stage_names[:6], mk[:-1], mk[1:]):
                    sums[s] += a.elapsed_time(b)
            else:
                sums["preprocess_bwd"] += mk[0].elapsed_time(mk[1])
                sums["allreduce"] += mk[1].elapsed_time(mk[2]) + mk[3].elapsed_time(mk[4])
                sums["adam"] += mk[2].elapsed_time(mk[3])
                if args.density_every:
                    sums["density"] += mk[4].elapsed_time(mk[5])
        return {s: sums[s] / steps for s in stage_names}

    # per-stage means: with several streams the views' stages overlap (their intervals would
    # include other views' kernels), so they come from a serial pass instead: the same steps
    # with every stage of every view in order on one stream, right after the timed region
    per_step = stage_means(record, args.steps)
    serial_steps = 0
    if serial_pass:
        serial_steps = args.serial_steps
        pool2 = [torch.cuda.Event(enable_timing=True) for _ in range(serial_steps * (7 * n_mine + 11))]
        rec2 = {"next": 0, "marks": [], "pool": pool2}
        barrier()
        for _ in range(serial_steps):
            one_step(dev_targets, rec2, hint_mode=hint_mode, serial=True)
        torch.cuda.synchronize()
        barrier()
        check_overflow("serial stage pass")
        per_step = stage_means(rec2, serial_steps)

    # ---- end-to-end through the public API with host buffers
    e2e = None
    if not args.no_e2e:
        copy_stream = torch.cuda.Stream(device=dev)
        tgt_events = [torch.cuda.Event() for _ in range(n_mine)]

        def e2e_step():
            # the step's targets go H2D on a copy stream (after the previous step released
            # the buffers); view j's loss waits for target j only, so the copies overlap the
            # earlier views' work
            copy_stream.wait_stream(stream)
            with torch.cuda.stream(copy_stream):
                for j, c in enumerate(rank_cams(step_no[0] + 1)):
                    targets_e2e[j].copy_(targets_host[c], non_blocking=True)
                    tgt_events[j].record(copy_stream)
            one_step(lambda j, c: targets_e2e[j], tgt_events=tgt_events, hint_mode=hint_mode)
            loss_host.copy_(loss, non_blocking=True)

        e2e_step()  # warm-up of the copy path
        restore()  # the pre-timing training state
        barrier()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(args.steps):
            e2e_step()
        e1.record(stream)
        torch.cuda.synchronize()
        barrier()
        check_overflow("e2e loop")
        e2e_ms = max_over_ranks(e0.elapsed_time(e1))
        e2e = {"value": args.views * args.steps / (e2e_ms / 1e3), "unit": UNIT,
               "h2d_bytes_per_step": int(targets_e2e[0].numel()) * args.views,
               "d2h_bytes_per_step": 4 * world}

    # ---- variants of the schedule (same work, same results; device-resident, timed alike)
    variants = None
    if not args.no_variants and not args.one_frame and not args.density_every:
        variants = {}
        runs = [("hinted" if args.hints == "none" else "unhinted", "camera" if args.hints == "none" else "none",
                 args.fixed_batch)]
        if not args.fixed_batch:
            runs.insert(0, ("fixed_batch", "slot", True))
        for name, mode, fixed in runs:
            restore()
            saved = args.fixed_batch
            args.fixed_batch = fixed  # rank_cams' default
            barrier()
            v0 = torch.cuda.Event(enable_timing=True)
            v1 = torch.cuda.Event(enable_timing=True)
            v0.record(stream)
            for _ in range(args.steps):
                one_step(dev_targets, hint_mode=mode)
            v1.record(stream)
            torch.cuda.synchronize()
            barrier()
            check_overflow(f"{name} loop")
            args.fixed_batch = saved
            vms = max_over_ranks(v0.elapsed_time(v1)) / args.steps
            variants[name] = {"value": round(args.views / (vms / 1e3), 3), "ms_per_step": round(vms, 3),
                              "batch": "views 4i mod 64 every step" if fixed else "views 4i + s mod 64 at step s",
                              "scheduling_hint": {"slot": "the frame's previous forward (same camera)",
                                                  "none": "none (work ordered by list length)",
                                                  "camera": "the camera's last forward"}[mode]}

    # ---- workload counters (not timed) for the roofline numerators: this rank's views of
    # the step after the timed loop's last
    stats = {"visible": 0, "num_keys": 0, "evals_fwd": 0, "evals_bwd": 0, "evals_slot": 0, "max_list": 0,
             "blended": 0, "evals_fwd_culled": 0, "evals_bwd_culled": 0}
    gs, n = S["gs"], S["n"]
    for rj, c in zip(S["rends"], rank_cams(step_no[0] + 1)):
        bgs.bgs_preprocess(gs, cam_structs_all[c], rj.frame)
        bgs.bgs_sort(rj.frame)
        bgs.bgs_render_fwd(rj.frame, rj.image, rj.final_T, rj.n_contrib)
        s = bgs.bgs_frame_stats(rj.frame, rj.n_contrib)
        for k2 in stats:
            if k2 == "max_list":
                stats[k2] = max(stats[k2], s.get(k2, 0))
            else:
                stats[k2] += s.get(k2, 0)

    # ---- shape statistics of the workload (reporting only, not timed): the
    # per-pixel walk lengths of view 0 and the local-density contrast the paper measures
    # (>= 100x between dense and sparse regions), rho at r = the scene's median
    # 8-NN distance (estimated from a 100k-point sample)
    shape = None
    if rank == 0:
        nc = S["rends"][0].n_contrib.to(torch.float64).flatten()
        qs = torch.quantile(nc[torch.randperm(nc.numel(), device=dev)[:1 << 20]],
                            torch.tensor([0.5, 0.99], dtype=torch.float64, device=dev)).tolist()
        from scipy.spatial import cKDTree

        mu = gen.segments(scene.theta, scene.n)["means"]
        sub = mu[gen.rng(77).choice(scene.n, min(scene.n, 100_000), replace=False)].astype(np.float64)
        r8 = float(np.median(cKDTree(sub).query(sub, k=9)[0][:, 8]) * (len(sub) / scene.n) ** (1.0 / 3.0))
        rho, _ = bgs.bgs_local_density(torch.from_numpy(mu.copy()).to(dev), r8)
        rq = torch.quantile(rho.to(torch.float64)[torch.randperm(rho.numel(), device=dev)[:1 << 20]],
                            torch.tensor([0.05, 0.5, 0.95, 0.99], dtype=torch.float64, device=dev)).tolist()
        shape = {"n_contrib_view0": {"median": qs[0], "p99": qs[1], "max": float(nc.max())},
                 "local_density_r": r8, "local_density_quantiles_p5_p50_p95_p99": rq,
                 "density_contrast_p99_over_p5": rq[3] / max(rq[0], 1.0)}

    # ---- max over ranks; the workload counters summed over ranks, per view of the step
    t = torch.tensor([ms_local], device=dev)
    views_counted = n_mine
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        keys = ("visible", "num_keys", "evals_fwd", "evals_bwd", "evals_slot", "blended", "evals_fwd_culled",
                "evals_bwd_culled")
        tt = torch.tensor([float(stats[k]) for k in keys] + [float(n_mine)], device=dev, dtype=torch.float64)
        dist.all_reduce(tt)
        for k, v_ in zip(keys, tt.tolist()):
            stats[k] = int(v_)
        views_counted = int(tt[-1].item())
    ms_total = float(t.item())
    ms_step = ms_total / args.steps
    value = args.views / (ms_step / 1e3)

    if rank != 0:
        return
    peaks, peaks_src = load_peaks()
    clocks = clk.summary()
    sm_mhz_max = float(peaks.get("sm_max_mhz", 1965.0))
    fp32_peak = 148 * FP32_LANES_PER_SM * sm_mhz_max * 1e6 / 1e12  # T lane-ops/s
    hbm = float(peaks.get("hbm_gbs", 6650.0))
    steps_views = n_mine  # views per step on rank 0 (its per-launch stage times)
    roof = {}
    # per-view numerators: averages over every rank's views of one step
    V = stats["visible"] / views_counted
    K = stats["num_keys"] / views_counted
    Ef, Eb, Ebl = (stats["evals_fwd"] / views_counted, stats["evals_bwd"] / views_counted,
                   stats["blended"] / views_counted)
    # what the blend kernels evaluate: list entries whose alpha >= 1/255 box reaches the
    # pixel's warp block (the exact skip of the rest)
    Efc, Ebc = stats["evals_fwd_culled"] / views_counted, stats["evals_bwd_culled"] / views_counted
    frame_v = S["rends"][0].views()
    passes = frame_v.sort_passes

    def frac(stage, achieved, peak, unit, bound, **extra):
        roof[stage] = {"bound": bound, "achieved": achieved, "peak": peak, "unit": unit,
                       "frac": achieved / peak if peak else None, "ms_per_launch": per_step[stage] / steps_views,
                       **extra}

    def per_launch(stage):
        return max(per_step[stage] / steps_views / 1e3, 1e-12)  # seconds (0 with --no-stage-events)

    if batch_pre:  # per launch of <= 16 views: theta's geometry 44 B per Gaussian + SH 192 B per Gaussian
        # some view sees (>= V: counted as V) once; per view radius + tiles_touched 8 B per Gaussian and
        # depth 4 + rect 8 + record 48 + clamp bits 1 + zeroed blend-gradient slots 48 per visible
        pre_launches = -(-steps_views // 16)
        pre_bytes = (44 * n + 192 * V) * pre_launches + (8 * n + 109 * V) * steps_views
        frac("preprocess", pre_bytes / max(per_step["preprocess"] / 1e3, 1e-12) / 1e9, hbm, "GB/s", "hbm")
        roof["preprocess"]["ms_per_launch"] = per_step["preprocess"] / pre_launches
        roof["preprocess"]["views_per_launch"] = min(16, steps_views)
    else:
        frac("preprocess", (16 * n + 268 * V) / per_launch("preprocess") / 1e9, hbm, "GB/s", "hbm")
    # sort: the algorithmic bytes of the path that runs
    if frame_v.sort_mode == 1:  # 64-bit onesweep reference: dup 12 + hist 8 + 24/pass per key, rects 20/visible
        sort_bytes, sort_def = (12 + 8 + 24 * passes) * K + 20 * V, "(12 + 8 + 24 p) B per key + 20 B per visible"
    elif args.sort_path == "radix_split":
        sort_bytes = 92 * V + (8 + 16 * (passes - 4)) * K
        sort_def = "92 B per visible (depth sort) + (8 + 16 per tile pass) B per key"
    else:  # depth sort of the visible Gaussians + the values written once by the direct split
        sort_bytes, sort_def = 92 * V + 4 * K, "92 B per visible + 4 B per key (SURVEY §8(d) a5 alternative, lower end)"
    frac("sort", sort_bytes / per_launch("sort") / 1e9, hbm, "GB/s", "hbm", work=sort_def)
    # blend: SURVEY §8(d) lane-ops per (pixel, list entry) pair by outcome over E_f / E_b (each
    # pixel's walk to its early stop, plain, before the exact block cull), and beside it the
    # same per-outcome counts over the pairs the kernels evaluate after the cull
    fwd_ops = OPS_FWD_BLENDED * Ebl + OPS_SKIPPED * (Ef - Ebl)
    bwd_ops = OPS_BWD_BLENDED * Ebl + OPS_SKIPPED * (Eb - Ebl)
    hw = _ncu_hw(args.config)
    for stage, ops, ops_c in (("render_fwd", fwd_ops, OPS_FWD_BLENDED * Ebl + OPS_SKIPPED * (Efc - Ebl)),
                              ("blend_bwd", bwd_ops, OPS_BWD_BLENDED * Ebl + OPS_SKIPPED * (Ebc - Ebl))):
        extra = {"work": f"SURVEY 8(d): {OPS_FWD_BLENDED if stage == 'render_fwd' else OPS_BWD_BLENDED} lane-ops "
                         f"per blended pair + {OPS_SKIPPED} per skipped pair over the plain walk",
                 "frac_after_cull": ops_c / per_launch(stage) / 1e12 / fp32_peak}
        if hw.get(stage):
            extra.update(hw[stage])
        frac(stage, ops / per_launch(stage) / 1e12, fp32_peak, "T lane-ops/s", "alu", **extra)
    if fused:  # a10 + a11: theta 236 read + 708 written (theta, m, v) + m, v 472 read per Gaussian, + per
        # (view, visible Gaussian) blend gradients 36 + radius 4 + clamp bits 1; radius 4 per (view, culled)
        pb_bytes = 1416 * n + (37 * V + 4 * n) * steps_views
        frac("preprocess_bwd", pb_bytes / max(per_step["preprocess_bwd"] / 1e3, 1e-12) / 1e9, hbm, "GB/s", "hbm")
        roof["preprocess_bwd"]["ms_per_launch"] = per_step["preprocess_bwd"]
        roof["preprocess_bwd"]["fused_with_adam"] = True
    elif args.one_frame:  # per view: theta 236 + blend grads 36 + grad RMW 472 per visible Gaussian
        frac("preprocess_bwd", 744 * V / per_launch("preprocess_bwd") / 1e9, hbm, "GB/s", "hbm")
    else:  # batched over the rank's views: theta 236 + grad 236 written (assigned) or 472 (read-modify-
        # written) per Gaussian once, + per (view, visible Gaussian) the blend gradients 36 + radius 4 + clamp
        # bits 1; radius 4 per (view, culled)
        pb_bytes = (472 if assign else 708) * n + (37 * V + 4 * n) * steps_views
        frac("preprocess_bwd", pb_bytes / max(per_step["preprocess_bwd"] / 1e3, 1e-12) / 1e9, hbm, "GB/s", "hbm")
        roof["preprocess_bwd"]["ms_per_launch"] = per_step["preprocess_bwd"] / -(-steps_views // 16)
    if not fused:
        # theta, m, v read + written and grad read: 1652 B per Gaussian, + 236 with grad zeroed (not assigned)
        adam_bytes = ((1652 if assign else 1888) * n / (world if sharded else 1)
                      + (236 * n if sharded and not assign else 0))
        roof["adam"] = {"bound": "hbm", "achieved": adam_bytes / max(per_step["adam"] / 1e3, 1e-12) / 1e9,
                        "peak": hbm, "unit": "GB/s", "ms_per_launch": per_step["adam"]}
        roof["adam"]["frac"] = roof["adam"]["achieved"] / hbm
    for k2, v2 in roof.items():
        assert v2["frac"] is None or v2["frac"] <= 1.5, f"roofline fraction of {k2} above 1: {v2}"
    # the dominant KERNEL: stages that are one kernel launch (the sort stage is 13 kernels;
    # it is reported in stages_roofline)
    dom = max((s for s in roof if s != "sort"), key=lambda s: per_step[s])
    traffic = None
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as f:
            # ncu_traffic.json is captured on the garden scene (tools/profile_round.sh)
            traffic = json.load(f).get(dom) if args.config == "garden" else None
    except Exception:
        pass
    d = roof[dom]
    roofline = {"bound": d["bound"], "achieved": round(d["achieved"], 3), "peak": round(d["peak"], 3),
                "unit": d["unit"], "frac": round(d["frac"], 4), "traffic": traffic, "kernel": dom,
                "peak_source": f"{peaks_src} (FP32: 148 SMs x 128 lanes x {sm_mhz_max:.0f} MHz)"
                if d["bound"] == "alu" else f"{peaks_src} MEASURED_PEAKS.json hbm_gbs"}
    for k2 in ("work", "frac_after_cull", "hw_lane_op_frac", "smem_wavefront_frac", "hw_source"):
        if k2 in d:
            roofline[k2] = round(d[k2], 4) if isinstance(d[k2], float) else d[k2]
    cpu = None
    if world == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline(args)
    line = {
        "metric": METRIC, "value": round(value, 3), "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": round(ms_step, 3), "ms_per_view": round(ms_step / args.views, 4),
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f32",
        "data": f"synthetic (seeded {scene.name}-shaped scene, gen/; random-init parameters; targets = render of "
                "a perturbed copy)",
        "config": arm_config(scene, args, world),
        "clocks": clocks, "gpu_launches": int(launches), "roofline": roofline,
        "stages_ms_per_step": {k2: round(v2, 4) for k2, v2 in per_step.items()},
        "stages_timing": (f"serial pass: {serial_steps} steps after the timed region, every stage of every view in "
                          "order on one stream (the timed region overlaps views on "
                          f"{n_streams} streams and sorts on {args.sort_streams}, and records no stage events)"
                          if serial_steps else "the timed region's own stage events"),
        "stages_roofline": {k2: {kk: (round(vv, 4) if isinstance(vv, float) else vv) for kk, vv in v2.items()}
                            for k2, v2 in roof.items()},
        "workload": {"V_per_view": V, "K_per_view": K, "E_f_per_view": Ef, "E_b_per_view": Eb,
                     "E_f_culled_per_view": Efc, "E_b_culled_per_view": Ebc, "blended_per_view": Ebl,
                     "E_slot_over_E_f_culled": stats["evals_slot"] / max(1, stats["evals_fwd_culled"]),
                     "max_tile_list": stats["max_list"], "shape": shape},
        "e2e": e2e, "cpu_baseline": cpu,
        "schedule": {"batch": "views 4i mod 64 every step" if args.fixed_batch else
                     "rotating: step s renders views 4i + s mod 64 (each camera every 4 steps)",
                     "scheduling_hint": "each frame's previous forward (same camera)" if args.fixed_batch else
                     ("each view hinted by its camera's last forward (bgs_frame_save_hint / load_hint)"
                      if args.hints == "camera" else "none: each forward's work ordered by its tile list lengths"),
                     "sort_path": args.sort_path,
                     "sorts": (f"all views' a4-a6 first, over {args.sort_streams} streams" if args.sort_streams > 0
                               and not args.one_frame else "each view's a4-a6 inline before its forward"),
                     "plans": ("forward schedules built with the sorts, backward schedules beside the loss "
                               "(bgs_render_fwd_plan / bgs_blend_bwd_plan)" if plan_ahead else "inline")},
        "variants": variants,
        "nccl": (nccl_summary() if world > 1 and os.environ.get("BGS_DIST_BACKEND", "nccl") == "nccl" else None),
        "density": None if not args.density_every else {
            "every": args.density_every, "r": round(float(dens_prm.r), 6), "events_timed_and_e2e": dens_log,
            "n_final": S["n"]},
    }
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------- oracle
# The oracle (oracle/bgs_oracle.cpp) as it stands -- the plain CPU program, OpenMP over
# independent units with fixed-order reductions -- timed on this host's cores.  Only here
# (the cpu_baseline leg and --impl reference) does bench.py execute oracle/.

ADAM_SLICE = 16  # Adam is timed on 1/16 of theta (its cost is exactly linear per element) and scaled


def _oracle_adam_seconds(n):
    """One O17 Adam step over 59 n elements: timed on the first 59 n / ADAM_SLICE, scaled."""
    import ctypes as C

    import oracle

    ns = max(1, n // ADAM_SLICE)
    r = np.random.default_rng(0)
    th, g, m, v = (r.standard_normal(59 * ns) for _ in range(4))
    v = np.abs(v)
    lr = np.array([1e-4, 5e-3, 1e-3, 0.05, 2.5e-3, 1.25e-4])
    p = [a.ctypes.data_as(C.c_void_p) for a in (th, g, m, v, lr)]
    t = time.perf_counter()
    oracle.lib().orc_adam(ns, *p, 0.9, 0.999, 1e-15, 1)
    return (time.perf_counter() - t) * n / ns


def _oracle_view_stages(scene, cam, dl, tile_mod=1, tile_phase=0):
    """One view through the oracle: O1-O9 preprocess, O10-O13 keys/sort/ranges over the whole
    scene, then the per-pixel walks (O14 forward, O15 backward) and O16 chain rule.  With
    tile_mod > 1 only the tile ROWS ty with ty % tile_mod == tile_phase are walked (a stratified
    1/tile_mod sample of the view's real tile lists, whole rows so that the oracle's parallel
    loops over rows / tile batches stay as busy as on the full view); the per-Gaussian parts of the backward
    (double preprocess + chain rule) are timed separately with every tile list emptied, so
    that only the walks are scaled.  Returns seconds per stage (walks already scaled)."""
    import oracle

    deg = scene.sh_degree
    T = {}
    t = time.perf_counter()
    pre = oracle.preprocess(scene.theta, scene.n, deg, cam)
    T["preprocess"] = time.perf_counter() - t
    t = time.perf_counter()
    srt = oracle.sort_keys(pre, cam)
    T["sort"] = time.perf_counter() - t
    ranges = srt["ranges"]
    if tile_mod > 1:
        ranges = ranges.copy()
        tiles_x = (cam.width + 15) // 16
        ranges[((np.arange(len(ranges)) // tiles_x) % tile_mod) != tile_phase] = 0
    sub = dict(srt, ranges=np.ascontiguousarray(ranges))
    t = time.perf_counter()
    oracle.render_fwd(pre, sub, cam)
    T["render_fwd"] = (time.perf_counter() - t) * tile_mod
    if tile_mod > 1:  # per-Gaussian part first (it also warms the allocator), then the sample
        empty = dict(srt, ranges=np.zeros_like(ranges))
        t = time.perf_counter()
        oracle.backward(scene.theta, scene.n, deg, cam, dict(pre=pre, srt=empty), dl)
        t_gauss = time.perf_counter() - t
    t = time.perf_counter()
    oracle.backward(scene.theta, scene.n, deg, cam, dict(pre=pre, srt=sub), dl)
    t_bwd = time.perf_counter() - t
    T["backward"] = t_gauss + max(0.0, t_bwd - t_gauss) * tile_mod if tile_mod > 1 else t_bwd
    T["K"] = srt["K"]
    return T


def cpu_baseline(args):
    """cpu_baseline of the main bench line (rank 0, N = 1): the oracle on ONE FULL view of
    the configured scene (camera 0: every Gaussian, every tile, every pixel; fwd + bwd) on all
    host cores, + the batch's Adam step amortised over its views; beside it BASELINE.json
    configs[0] (tiny: 4096 Gaussians, 128x128) fwd + bwd + Adam on one core."""
    import gen
    import oracle

    scene = gen.make(args.config)
    cam = scene.cameras[0]
    dl = gen.random_dl_dimage(0, cam.width, cam.height, scale=1e-6)
    cores = oracle.set_threads(0)
    T = _oracle_view_stages(scene, cam, dl)
    t_adam = _oracle_adam_seconds(scene.n)
    view_s = sum(v for k, v in T.items() if k != "K") + t_adam / args.views
    # tiny (configs[0]) on one core: preprocess -> sort -> fwd -> bwd -> Adam, the whole iteration
    tiny = gen.tiny()
    oracle.set_threads(1)
    tc = tiny.cameras[0]
    t = time.perf_counter()
    f = oracle.forward(tiny.theta, tiny.n, tiny.sh_degree, tc)
    b = oracle.backward(tiny.theta, tiny.n, tiny.sh_degree, tc, f, gen.random_dl_dimage(1, tc.width, tc.height))
    oracle.adam(tiny.theta, b["grad"], np.zeros(59 * tiny.n), np.zeros(59 * tiny.n), tiny.n,
                [1e-4, 5e-3, 1e-3, 0.05, 2.5e-3, 1.25e-4])
    tiny_s = time.perf_counter() - t
    oracle.set_threads(0)
    return {"value": round(1.0 / view_s, 6), "unit": UNIT, "cores": cores, "kind": "oracle",
            "sample": f"full scene, {cores} cores: 1 view (camera 0) of the {scene.name} scene, all {scene.n} "
                      f"Gaussians, {cam.width}x{cam.height}, K = {T['K']} keys, fwd+bwd {view_s - t_adam / args.views:.2f} s "
                      f"+ Adam over 59N ({t_adam:.2f} s per batch, timed on 1/{ADAM_SLICE} of theta and scaled) / "
                      f"{args.views} views",
            "stages_s": {k: round(v, 3) for k, v in T.items() if k != "K"},
            "tiny_1core": {"config": "tiny: 4096 Gaussians, 128x128, SH 3 (BASELINE.json configs[0])",
                           "fwd_bwd_adam_s": round(tiny_s, 4), "cores": 1},
            "cpu": _cpu_model()}


def _cpu_model():
    try:
        for ln in open("/proc/cpuinfo"):
            if ln.startswith("model name"):
                return ln.split(":", 1)[1].strip() + f" ({os.cpu_count()} logical cores on host)"
    except Exception:
        pass
    return f"{os.cpu_count()} logical cores"


def run_reference(args, rank, world):
    """The reference arm of this tier: the oracle, as it stands, on this host's cores, on the
    same config / metric / unit as our arm.  Each step is a bounded sample of one step's
    workload: one full view of the scene (camera of that step, every Gaussian) through the
    per-Gaussian stages and the sort, a stratified 1/tile_mod of its tile rows (rotating with
    the step, so 8 steps cover every tile once) through the per-pixel walks, scaled to the whole
    view, and the batch's Adam; the step's time = views x (one view) + Adam."""
    if rank != 0:
        return
    import gen
    import oracle

    tile_mod = 8
    scene = gen.make(args.config)
    cams = [scene.cameras[v] for v in batch_views(args.views, len(scene.cameras))]
    cores = oracle.set_threads(0)
    cam0 = cams[0]
    dl = gen.random_dl_dimage(0, cam0.width, cam0.height, scale=1e-6)
    t_adam = _oracle_adam_seconds(scene.n)

    def step(i):
        T = _oracle_view_stages(scene, cams[i % len(cams)], dl, tile_mod, i % tile_mod)
        return args.views * sum(v for k, v in T.items() if k != "K") + t_adam

    for i in range(args.warmup):
        step(i)
    sec = sum(step(args.warmup + i) for i in range(args.steps)) / args.steps
    value = args.views / sec
    line = {"impl": "reference", "metric": METRIC, "value": round(value, 6), "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(sec * 1e3, 3),
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64/f32",
            "data": "synthetic", "config": arm_config(scene, args, world),
            "cpu_baseline": {"value": round(value, 6), "unit": UNIT, "cores": cores, "kind": "oracle",
                             "sample": f"each step: one full view of the {scene.name} scene ({scene.n} Gaussians, "
                                       f"the step's camera) through preprocess, keys and sort on {cores} cores; "
                                       f"the per-pixel blend walks (fwd + bwd) on a stratified 1/{tile_mod} of "
                                       f"its tile rows, scaled x{tile_mod}; x{args.views} views + one Adam over 59N "
                                       f"(timed on 1/{ADAM_SLICE} of theta, scaled); supplied dL/dimage",
                             "cpu": _cpu_model()},
            "e2e": {"value": round(value, 6), "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def main():
    args = parse()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        run_reference(args, rank, world)
        return
    if world > 1:
        import torch
        import torch.distributed as dist

        backend = os.environ.get("BGS_DIST_BACKEND", "nccl")
        torch.cuda.set_device(_device_index(local_rank))
        if backend == "nccl":
            # NCCL's own log (init, topology, NVLS) to a per-process file; rank 0 quotes the
            # lines that confirm the ranks, transport and algorithm in its JSON line
            os.environ.setdefault("NCCL_DEBUG", "INFO")
            os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT,GRAPH,NVLS")
            os.environ.setdefault("NCCL_DEBUG_FILE", "/tmp/bgs_nccl.%h.%p.log")
            dist.init_process_group("nccl", device_id=torch.device("cuda", _device_index(local_rank)))
        else:  # test-only: several ranks sharing one GPU (NCCL refuses duplicate GPUs)
            dist.init_process_group(backend)
    try:
        run_ours(args, rank, world, local_rank)
    finally:
        if world > 1:
            import torch.distributed as dist

            dist.destroy_process_group()


if __name__ == "__main__":
    main()
