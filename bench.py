#!/usr/bin/env python
"""bench.py — FCFS hot-path throughput on B200 (BASELINE.json metric: Fourier coeff.vertex
terms/sec, Gterm/s, and % of tensor peak, 1/2/4/8 B200).

One STEP = one pass of the whole hot path over one batch:
  a1 fcfs_vertices_from_rects (rects -> signed corners + area)  then
  a2-a5 fcfs_coeffs_batched   (twiddles + contraction + axes/DC + pupil epilogue).
Default workload = BASELINE.json configs[2] ("c3"): 4096 clips per GPU, T = 2048, ~1200
lines/clip, ~4.8k corners/clip, pupil radius 27.22 (2337 coefficients/clip), split-TF32.
Multi-GPU (torchrun): clips are sharded — every rank runs its own 4096 clips (weak
scaling, no data-path collective); time = max over ranks (all_reduce MAX).

terms = sum over clips of W_out x K_clip.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

from paper_1010_5562_b200 import inputs  # noqa: E402


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="c3", choices=["c1", "c2", "c3", "c4", "c5", "layout", "haar"],
                    help="layout: c3-style lines over a tiles x tiles layout of T=2048 tiles, chopped into tiles "
                         "on the GPU (fcfs_chop_rects) and transformed as one batch (the paper's flow, P:1060-1062)")
    ap.add_argument("--tiles", type=int, default=64, help="layout: tiles per side")
    ap.add_argument("--haar-tiles", type=int, default=16, help="haar: tiles per side (T=1024 tiles)")
    ap.add_argument("--prec", default=None, choices=["fp64", "tf32x3", "f16x3"])
    ap.add_argument("--clips", type=int, default=4096, help="c3 clips per GPU")
    ap.add_argument("--shard", default="rows", choices=["rows", "peers", "vblock"],
                    help="single-clip configs (c1, c2, c4, c5) on N > 1 GPUs: frequency rows + all_gather, "
                         "frequency rows stored by the epilogue into every rank's window over NVLink "
                         "(fcfs_coeffs_rows_to_peers), or vertex blocks + reduce_scatter")
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--route", default=None, choices=["auto", "gemm", "fft"],
                    help="single-clip configs: fcfs_options.route (default: the library's cost model)")
    ap.add_argument("--form", default=None, choices=["auto", "edge", "corner", "lattice"],
                    help="batched split precisions: fcfs_options.form (default: the library's choice)")
    ap.add_argument("--input", default="rects", choices=["rects", "polygons"],
                    help="a1 input: rects (fcfs_vertices_from_rects) or the same rects as 4-vertex polygon "
                         "lists (fcfs_vertices_from_polygons; workloads with one group per rect)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=12.0, help="target CPU oracle sample time")
    ap.add_argument("--e2e-split", type=int, default=8, help="sub-batches of the pipelined end-to-end measurement")
    ap.add_argument("--no-small", action="store_true",
                    help="small single clips (c1): the general extraction + coefficient path instead of the "
                         "one-launch fcfs_small_clip latency path replayed as a CUDA graph")
    ap.add_argument("--no-graph", action="store_true",
                    help="single clips on the lattice-FFT route: time the host-synchronising API calls instead of "
                         "the sync-free pipeline (fcfs_vertices_from_rects_async + fcfs_coeffs_async) replayed as "
                         "a CUDA graph")
    ap.add_argument("--no-extra", action="store_true",
                    help="skip the extra lines (c4 / c5 FP64, c4 split-TF32) of the default c3 run")
    return ap.parse_args()


def _free_port():
    import socket
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def spawn_ranks(args):
    """--gpus N without a torchrun environment: re-exec this command under torch.distributed.run with N
    ranks (one process per GPU, rendezvous on 127.0.0.1)."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr=127.0.0.1", f"--master-port={_free_port()}", os.path.abspath(__file__)] + sys.argv[1:]
    os.execv(sys.executable, cmd)


EXTRAS = (("c4", "fp64", None), ("c5", "fp64", None), ("c4", "tf32x3", None), ("c4", "fp64", "gemm"))


def run_extras(args):
    """The default c3 run also measures the FP64 single-clip configs (lattice-FFT route, the default),
    c4 split-TF32 and c4 FP64 on the row-bucket DMMA GEMM route (the FP64 tensor-core roofline), each in a
    child bench.py process (its own plans, clocks, roofline and sampled oracle baseline); their lines are
    embedded under "extra"."""
    out = {}
    for cfg, prec, route in EXTRAS:
        cmd = [sys.executable, os.path.abspath(__file__), "--config", cfg, "--prec", prec, "--steps",
               str(min(args.steps, 5)), "--warmup", "3", "--no-e2e", "--no-extra", "--cpu-seconds", "4"]
        if route:
            cmd += ["--route", route]
        if prec != "fp64" or route:
            cmd.append("--no-cpu-baseline")         # the oracle does not depend on the precision / route
        try:
            r = subprocess.run(cmd, capture_output=True, text=True, timeout=600,
                               env=dict(os.environ, WORLD_SIZE="1", RANK="0", LOCAL_RANK="0"))
            lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
            d = json.loads(lines[-1]) if lines else {"error": (r.stderr or "no output")[-400:]}
        except Exception as ex:   # a failed extra must not lose the main line
            d = {"error": repr(ex)[:400]}
        for k in ("e2e", "metric", "unit", "higher_is_better", "vs_baseline", "data", "n_gpus"):
            d.pop(k, None)
        out[f"{cfg}_{prec}" + (f"_{route}" if route else "")] = d
    return out


def load_peaks():
    try:
        return json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))), "measured"
    except Exception:
        return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0, "sm_max_mhz": 1965.0}, \
            "fallback"


def workload(cfg, seed, rank, clips, tiles=64):
    if cfg == "layout":
        T = 2048
        lay = inputs.layout(seed + rank, T=T, tiles_x=tiles, tiles_y=tiles)
        r2 = inputs.pupil_r2(T)
        M = int(math.floor(math.sqrt(r2)))
        # clip_ptr is a placeholder of the tile count (the tiles are made on the GPU by the chop step)
        wl = inputs.Workload("layout", T, M, M, r2, lay.rects, None, np.zeros(tiles * tiles + 1, np.int64),
                             ("tf32x3",))
        wl.layout = lay
        return wl
    if cfg == "c3":
        # weak scaling: each rank its own clip range (seed streams (seed, clip) with clip offset by rank)
        T = 2048
        rects = np.concatenate([inputs.c3_clip(seed, rank * clips + b, T) for b in range(clips)])
        cp = np.arange(0, clips + 1, dtype=np.int64) * 1200
        r2 = inputs.pupil_r2(T)
        M = int(math.floor(math.sqrt(r2)))
        return inputs.Workload("c3", T, M, M, r2, rects, None, cp, ("tf32x3",))
    return inputs.make(cfg, seed=seed + rank)


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    def __init__(self, index):
        self.index = index
        self.rows = []
        self.proc = None

    def __enter__(self):
        q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
             "clocks_event_reasons.sw_power_cap")
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={q}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([c.strip() for c in line.split(",")])

    def __exit__(self, *a):
        if self.proc:
            time.sleep(0.15)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except Exception:
                self.proc.kill()

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = set()
        for r in self.rows:
            for i, n in enumerate(names):
                if len(r) > 4 + i and r[4 + i].lower().startswith("active"):
                    reasons.add(n)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(self.rows)}


def cpu_baseline(wl, target_s, prec, one_core=True):
    """The oracle as it stands (extraction + direct sums), timed on a bounded sample of the workload.

    Extraction and coefficients are timed separately, on all host cores (the oracle's
    OpenMP coefficient loop; its extraction is serial) and, when one_core, again on one core (the
    paper's single-threaded setup).  Batched clips: whole clips (all coefficients) until
    ~target_s.  One clip: the full extraction plus a fixed random sample of coefficients, extrapolated
    to the full window (t = t_extract + t_sample x W / sample)."""
    import oracle
    cores = oracle.max_threads()
    ms, ns = oracle.window(wl.M, wl.N, wl.r2)
    W = len(ms)
    chop_s = 0.0
    if getattr(wl, "layout", None) is not None:
        lay = wl.layout
        t0 = time.perf_counter()
        ch = oracle.chop_rects(lay.rects, lay.T, lay.tiles_x, lay.tiles_y)
        chop_s = time.perf_counter() - t0
        wl = inputs.Workload("layout tiles", wl.T, wl.M, wl.N, wl.r2, ch["rects"], None, ch["tile_ptr"], ())

    def extract_clip(b):
        r0, r1 = wl.clip_rect_range(b % wl.B)
        gp = None
        if wl.group_ptr is not None:
            g0, g1 = (wl.clip_ptr[b], wl.clip_ptr[b + 1]) if wl.clip_ptr is not None else (0, len(wl.group_ptr) - 1)
            gp = wl.group_ptr[g0:g1 + 1] - wl.group_ptr[g0]
        t0 = time.perf_counter()
        e = oracle.extract(wl.rects[r0:r1], wl.T, gp)
        return e, time.perf_counter() - t0

    if wl.B == 1 and wl.R > 20000:
        # one huge clip: the whole extraction + a sample of the output set, extrapolated to all W outputs
        e, t_ex = extract_clip(0)
        K = e["K"]
        rng = np.random.default_rng(0)
        pick = rng.choice(W, size=min(W, 64), replace=False)
        t0 = time.perf_counter()
        oracle.coeffs(e["x"], e["y"], e["w"], e["area"][0], wl.T, ms[pick], ns[pick])
        t_c = (time.perf_counter() - t0) / len(pick)               # per coefficient, all cores
        terms = float(W) * K
        full = t_ex + t_c * W
        out = {"value": terms / full / 1e9, "unit": "Gterm/s", "cores": cores, "kind": "oracle",
               "sample": (f"1 clip: full extraction (K={K}) + {len(pick)} of {W} coefficients (seeded random), "
                          f"extrapolated to all {W}"),
               "extract_s": round(t_ex, 4), "coeffs_s_per_coef": t_c, "extrapolated_full_s": round(full, 2),
               "seconds": round(t_ex + t_c * len(pick), 3)}
        if one_core:
            p1 = pick[:16]
            t0 = time.perf_counter()
            oracle.coeffs(e["x"], e["y"], e["w"], e["area"][0], wl.T, ms[p1], ns[p1], nthreads=1)
            t_c1 = (time.perf_counter() - t0) / len(p1)
            full1 = t_ex + t_c1 * W
            out["one_core"] = {"value": terms / full1 / 1e9, "unit": "Gterm/s", "cores": 1,
                               "sample": f"the same extraction + {len(p1)} coefficients on one core, extrapolated",
                               "coeffs_s_per_coef": t_c1, "extrapolated_full_s": round(full1, 2)}
        return out

    def run(nthreads, budget):
        terms = 0
        t_ex = t_co = 0.0
        n = 0
        t0 = time.perf_counter()
        while True:
            e, te = extract_clip(n)
            tc0 = time.perf_counter()
            oracle.coeffs(e["x"], e["y"], e["w"], e["area"][0], wl.T, ms, ns, nthreads=nthreads)
            t_co += time.perf_counter() - tc0
            t_ex += te
            terms += W * e["K"]
            n += 1
            if time.perf_counter() - t0 > budget or n >= wl.B:
                break
        return terms, n, t_ex, t_co

    terms, n, t_ex, t_co = run(0, target_s)
    dt = t_ex + t_co + chop_s * n / max(wl.B, 1)
    sample = f"{n} clips (extraction + all {W} coefficients each)"
    if chop_s:
        sample += f"; + the host chop of the whole layout ({chop_s:.2f} s) charged pro rata"
    out = {"value": terms / dt / 1e9, "unit": "Gterm/s", "cores": cores, "kind": "oracle", "sample": sample,
           "seconds": round(dt, 3), "extract_s_per_clip": t_ex / n, "coeffs_s_per_clip": t_co / n}
    if one_core:
        terms1, n1, t_ex1, t_co1 = run(1, max(1.0, target_s / 3))
        dt1 = t_ex1 + t_co1 + chop_s * n1 / max(wl.B, 1)
        out["one_core"] = {"value": terms1 / dt1 / 1e9, "unit": "Gterm/s", "cores": 1,
                           "sample": f"{n1} clips on one core", "seconds": round(dt1, 3),
                           "extract_s_per_clip": t_ex1 / n1, "coeffs_s_per_clip": t_co1 / n1}
    return out


def run_reference(args, rank, world):
    """--impl reference: the CPU oracle (this tier's reference arm) on the same workload."""
    if rank != 0:
        return
    if args.config == "haar":
        # the oracle's continuous Haar transform (child-cell areas) on one chopped tile per step
        import oracle
        T, nt = 1024, args.haar_tiles
        lay = inputs.layout(args.seed, T=T, tiles_x=nt, tiles_y=nt, lines_per_tile=300)
        ch = oracle.chop_rects(lay.rects, T, nt, nt)
        vals = []
        for i in range(args.warmup + args.steps):
            a, b = ch["tile_ptr"][i % (nt * nt)], ch["tile_ptr"][i % (nt * nt) + 1]
            e = oracle.extract(ch["rects"][a:b], T)
            t0 = time.perf_counter()
            oracle.haar(e["x"], e["y"], e["w"], T)
            if i >= args.warmup:
                vals.append(T * T / (time.perf_counter() - t0) / 1e9)
        v = statistics.median(vals)
        line = {"impl": "reference", "metric": "haar_coefficients_per_sec", "value": v, "unit": "Gcoef/s",
                "n_gpus": 0, "steps": args.steps, "warmup": args.warmup, "higher_is_better": True, "scaling": "weak",
                "vs_baseline": None, "dtype": "exact integer areas (int64 / int128)", "data": "synthetic",
                "config": {"workload": f"haar: one T={T} tile per step of the {nt}x{nt}-tile layout"},
                "cpu_baseline": {"value": v, "unit": "Gcoef/s", "cores": 1, "kind": "oracle",
                                 "sample": "one tile per step, oracle_haar single thread"},
                "e2e": {"value": v, "unit": "Gcoef/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
        print(json.dumps(line), flush=True)
        return
    wl = workload(args.config, args.seed, 0, args.clips, args.tiles)
    prec = args.prec or ("tf32x3" if args.config in ("c3", "layout") else "fp64")
    per_step = max(2.0, min(20.0, 60.0 / max(1, args.steps + args.warmup)))
    for _ in range(args.warmup):
        cpu_baseline(wl, per_step / 4, prec, one_core=False)
    vals = []
    last = None
    for _ in range(args.steps):
        last = cpu_baseline(wl, per_step, prec, one_core=False)
        vals.append(last["value"])
    v = statistics.median(vals)
    line = {"impl": "reference", "metric": "fourier_coeff_vertex_terms_per_sec", "value": v, "unit": "Gterm/s",
            "n_gpus": 0, "steps": args.steps, "warmup": args.warmup, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f80 (x87 long double)", "data": "synthetic",
            "config": config_dict(args, wl, prec, world),
            "cpu_baseline": {"value": v, "unit": "Gterm/s", "cores": last["cores"], "kind": "oracle",
                             "sample": last["sample"]},
            "e2e": {"value": v, "unit": "Gterm/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def edge_counts(vp, K, cptr_h):
    """Inner dimension of the batched split-TF32 kernel in edge form (edges.cu): per clip, the corners
    that head a pair or stay single.  A link joins corners k-1, k of one clip with equal y and
    opposite weights; chains of links pair up at even positions.  Counted here on the host from the
    extracted corners (outside the timed region) for the roofline's algorithmic flops."""
    y = vp.y[:K].cpu().numpy().astype(np.int64)
    w = vp.w[:K].cpu().numpy().astype(np.int64)
    k = np.arange(K)
    first = np.zeros(K, bool)
    first[cptr_h[:-1][cptr_h[:-1] < K]] = True
    link = np.zeros(K, bool)
    link[1:] = (y[1:] == y[:-1]) & (w[1:] == -w[:-1])
    link &= ~first
    start = np.maximum.accumulate(np.where(~link, k, 0))
    emit = ((k - start) % 2) == 0
    clip = np.searchsorted(cptr_h, k, side="right") - 1
    return np.bincount(clip, weights=emit, minlength=len(cptr_h) - 1).astype(np.float64)


def traffic_for(cfg, prec, route=""):
    """dram read+write bytes per launch of the dominant kernel (or, for the FFT route, of the contract
    stage's kernels) from the committed ncu --set full captures (profiles/traffic.json), or None when
    no capture matches this config / precision / route."""
    try:
        t = json.load(open(os.path.join(ROOT, "profiles", "traffic.json")))
        return t.get(f"{cfg}/{prec}" + (f"/{route}" if route else ""))
    except Exception:
        return None


def config_dict(args, wl, prec, world):
    W = inputs.window_count(wl.M, wl.N, wl.r2)
    d = {"workload": f"{wl.name}: T={wl.T}, {wl.B} clip(s)/GPU, R={wl.R} rects/GPU, window |m|,|n|<={wl.M}"
                     + (f" pupil r2={wl.r2:.2f}" if wl.r2 >= 0 else "") + f", W_out={W}/clip",
         "T": wl.T, "clips_per_gpu": wl.B, "rects_per_gpu": wl.R, "M": wl.M, "N": wl.N, "W_out": W,
         "precision": prec,
         "parallelism": (f"clip-sharded x{world}" if wl.B > 1 else
                         (f"{args.shard}-sharded x{world}" if world > 1 else "single GPU")),
         "l2": "flushed between steps (512 MiB write, outside the timed events)"}
    if getattr(args, "input", "rects") == "polygons":
        d["input"] = "each rect as a clockwise 4-vertex polygon (fcfs_vertices_from_polygons)"
    if getattr(wl, "layout", None) is not None:
        lay = wl.layout
        d["workload"] = (f"layout: {lay.tiles_x}x{lay.tiles_y} tiles of T={lay.T} ({lay.tiles_x * lay.T}^2 grid), "
                         f"R={wl.R} c3-style lines; step = chop into tiles + extraction + pupil coefficients "
                         f"(|m|,|n|<={wl.M}, r2={wl.r2:.2f}, W_out={W}/tile)")
        d["tiles"] = lay.tiles_x * lay.tiles_y
    return d


def bench_haar(args, rank, world, dev):
    """NEXT-4: the continuous Haar transform of a chopped layout (T = 1024 tiles, the paper's 1024 nm
    tiles at 1 nm): one step = chop + batched extraction + fcfs_haar of every tile."""
    import torch
    import torch.distributed as dist
    from paper_1010_5562_b200 import fcfs
    T = 1024
    nt = args.haar_tiles
    lay = inputs.layout(args.seed + rank, T=T, tiles_x=nt, tiles_y=nt, lines_per_tile=300)
    rects = torch.from_numpy(lay.rects).to(dev)
    chop = fcfs.ChopPlan(lay.rects.shape[0], T, nt, nt, device=dev)
    n_p = chop.run(rects)
    B = nt * nt
    vp = fcfs.VerticesPlan(n_p, T, n_p, B, 1, grouped=False, device=dev)
    hp = fcfs.HaarPlan(B, T, device=dev)

    def step():
        chop.run(rects)
        k = vp.run(chop.out[:n_p], None, chop.tile_ptr)
        return hp.run(vp.x[:k], vp.y[:k], vp.w[:k], vp.area, vp.corner_ptr)
    for _ in range(args.warmup):
        step()
    flush = torch.empty(512 * 1024 * 1024, dtype=torch.uint8, device=dev)
    fcfs.profile_enable(True)
    fcfs.profile_read()
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    launches0 = fcfs.kernel_launches()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    with ClockSampler(int(os.environ.get("LOCAL_RANK", "0"))) as clk:
        for i in range(args.steps):
            evs[i][0].record()
            step()
            evs[i][1].record()
            flush.fill_(i & 0xff)
        torch.cuda.synchronize()
    launches = fcfs.kernel_launches() - launches0
    stages = fcfs.profile_read()
    fcfs.profile_enable(False)
    total_ms = sum(a.elapsed_time(b) for a, b in evs)
    t = torch.tensor([total_ms], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms = float(t.item()) / args.steps
    coefs = float(B) * T * T
    value = coefs * world / (ms / 1e3) / 1e9
    h_ms = stages["contract"][0] / args.steps
    peaks, src = load_peaks()
    ach = coefs * 8.0 / (h_ms / 1e3) / 1e9        # algorithmic bytes: the 8-byte coefficient written once
    roof = {"bound": "hbm", "achieved": round(ach, 1), "peak": peaks["hbm_gbs"], "unit": "GB/s",
            "frac": round(ach / peaks["hbm_gbs"], 4), "traffic": None, "kernel": "fcfs_haar (band sweep: k_haar_yptr + k_haar_band)",
            "alg_bytes_per_launch": coefs * 8.0, "kernel_ms_per_launch": round(h_ms, 4),
            "stage_ms_per_step": {k: round(v[0] / args.steps, 4) for k, v in stages.items()},
            "peak_source": f"{src} HBM copy bandwidth"}
    if rank == 0:
        line = {"metric": "haar_coefficients_per_sec", "value": round(value, 3), "unit": "Gcoef/s", "n_gpus": world,
                "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms, 4), "higher_is_better": True,
                "scaling": "weak", "vs_baseline": None, "dtype": "f64 (exact dyadic values from int64 numerators)",
                "data": "synthetic",
                "config": {"workload": f"haar: {nt}x{nt} tiles of T={T}, c3-style lines (300 per tile), chop + "
                                       f"extraction + continuous Haar transform (J=10, all T^2 coefficients per tile)",
                           "tiles": B, "T": T, "pieces": n_p, "l2": "flushed between steps"},
                "roofline": roof, "clocks": clk.summary(), "gpu_launches": int(launches), "e2e": None}
        if world == 1 and not args.no_cpu_baseline:
            import oracle
            ch = oracle.chop_rects(lay.rects, T, nt, nt)
            a, b = ch["tile_ptr"][0], ch["tile_ptr"][1]
            e = oracle.extract(ch["rects"][a:b], T)
            t0 = time.perf_counter()
            oracle.haar(e["x"], e["y"], e["w"], T)
            dt = time.perf_counter() - t0
            line["cpu_baseline"] = {"value": T * T / dt / 1e9, "unit": "Gcoef/s", "cores": 1, "kind": "oracle",
                                    "sample": f"1 tile (K={e['K']}), oracle_haar (child-cell areas, single thread)",
                                    "seconds": round(dt, 3)}
        print(json.dumps(line), flush=True)


def main():
    args = parse()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        spawn_ranks(args)                          # does not return
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        raise SystemExit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}")
    if args.impl == "reference":
        run_reference(args, rank, world)
        return

    import torch
    import torch.distributed as dist
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if args.config == "haar":
        if world > 1:
            dist.init_process_group("nccl", device_id=dev)
        from paper_1010_5562_b200 import fcfs as _f
        _f.device_check()
        bench_haar(args, rank, world, dev)
        if world > 1:
            dist.destroy_process_group()
        return
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    from paper_1010_5562_b200 import fcfs

    fcfs.device_check()
    prec = args.prec or ("tf32x3" if args.config in ("c3", "layout") else "fp64")
    wl = workload(args.config, args.seed, rank, args.clips, args.tiles)
    layout = "pupil" if wl.r2 >= 0 else "dense"
    W = inputs.window_count(wl.M, wl.N, wl.r2)

    # inputs resident in HBM (value) and pinned host copies (e2e)
    rects_h = torch.from_numpy(wl.rects).pin_memory()
    rects = rects_h.to(dev)
    gp = None if wl.group_ptr is None else torch.from_numpy(wl.group_ptr).to(dev)
    cp = None if wl.clip_ptr is None else torch.from_numpy(wl.clip_ptr).to(dev)
    mg = 1 if wl.group_ptr is None else int(np.diff(wl.group_ptr).max())
    G = wl.R if wl.group_ptr is None else len(wl.group_ptr) - 1
    small = None
    graph_launches = 0   # kernels per replay of a captured step (replays bypass the launch counter)
    if (wl.B == 1 and world == 1 and args.input == "rects" and args.config != "layout" and not args.no_small
            and fcfs.SmallClipPlan.supported(wl.R, wl.T, wl.M, wl.N, wl.r2, layout, G, mg)):
        # latency path: a1-a5 in one kernel launch with no host sync (fcfs_small_clip), the step
        # captured once in a CUDA graph and replayed
        small = fcfs.SmallClipPlan(wl.R, wl.T, wl.M, wl.N, wl.r2, layout, prec, G=G, max_group=mg, device=dev)
        small.run(rects, gp)
        torch.cuda.synchronize()
        K_small = small.check()
        g_stream = torch.cuda.Stream(dev)
        graph = torch.cuda.CUDAGraph()
        lc0 = fcfs.kernel_launches()
        with torch.cuda.graph(graph, stream=g_stream):
            small.run(rects, gp, stream=g_stream)
        graph_launches = fcfs.kernel_launches() - lc0   # this library's kernels in one replay
        vp = None

        def extract():
            return K_small
    elif args.config == "layout":
        # layout -> tiles on the GPU, then the tiles' corners as one batch
        lay = wl.layout
        chop = fcfs.ChopPlan(wl.R, wl.T, lay.tiles_x, lay.tiles_y, device=dev)
        n_pieces = chop.run(rects)
        vp = fcfs.VerticesPlan(n_pieces, wl.T, n_pieces, wl.B, 1, grouped=False, device=dev)

        def extract():
            chop.run(rects)
            return vp.run(chop.out[:n_pieces], None, chop.tile_ptr)
    elif args.input == "polygons":
        if wl.group_ptr is not None:
            raise SystemExit("--input polygons needs a workload with one group per rect (c3, c4, c5)")
        ps = inputs.rects_as_polygons(wl.rects, wl.T, wl.clip_ptr)
        pvx, pvy = torch.from_numpy(ps.vx).to(dev), torch.from_numpy(ps.vy).to(dev)
        ppp = torch.from_numpy(ps.poly_ptr).to(dev)
        vp = fcfs.PolygonsPlan(ps.vx.shape[0], ps.P, wl.T, wl.B, device=dev)

        def extract():
            return vp.run(pvx, pvy, ppp, cp)
    elif wl.B == 1 and world > 1:
        # one clip on N GPUs: a1 sharded by lattice-row bands (fcfs_vertices_from_rects_band) and the
        # band lists all_gathered into the canonical list on every rank (dist.gather_corners)
        from paper_1010_5562_b200 import dist as fdist
        vp = None
        bandx = fdist.BandExtract(wl.R, wl.T, rank, world, G=G, max_group=mg, grouped=gp is not None, device=dev)
        gathered = {}

        def extract():
            x, y, w, k, a = fdist.gather_corners(*bandx.run(rects, gp))
            gathered.update(x=x, y=y, w=w, K=k, area=a)
            return k
    else:
        vp = fcfs.VerticesPlan(wl.R, wl.T, G, wl.B, mg, grouped=gp is not None, device=dev)

        def extract():
            return vp.run(rects, gp, cp)
    K = extract()
    cptr_h = vp.corner_ptr.cpu().numpy() if vp is not None else np.array([0, K], np.int64)
    kmax = int(np.diff(cptr_h).max()) if wl.B > 0 else 0
    if small is not None:
        plan = small

        def coeffs():
            graph.replay()
            return small.out
        out_bytes = small.out.numel() * small.out.element_size()
    elif wl.B > 1:
        plan = fcfs.BatchedPlan(wl.B, K, kmax, wl.T, wl.M, wl.N, wl.r2, layout, prec, device=dev, form=args.form,
                                sorted_y=True)   # corners from fcfs_vertices_from_* are y-sorted per clip

        def coeffs():
            return plan.run(vp.corner_ptr, vp.x[:K], vp.y[:K], vp.w[:K], vp.area)
        out_bytes = plan.out.numel() * plan.out.element_size()
    elif world > 1:
        # ... then each rank computes its shard with its own pre-built plan and the collective assembles
        # the full window (strong scaling): frequency rows + all_gather, or corner blocks (GEMM route) +
        # reduce_scatter + all_gather
        full_n = (2 * wl.M + 1) * (2 * wl.N + 1)

        class _P:
            out = torch.empty(full_n, dtype=torch.complex128 if prec == "fp64" else torch.complex64, device=dev)
        plan = _P()
        if args.shard == "rows":
            sharded = fdist.RowsSharded(wl.T, wl.M, wl.N, prec, rank, world, device=dev, route=args.route)
        elif args.shard == "peers":
            sharded = fdist.RowsPeers(wl.T, wl.M, wl.N, prec, rank, world, device=dev, route=args.route)
        else:
            sharded = fdist.VertexSharded(wl.T, wl.M, wl.N, prec, rank, world, device=dev)

        def coeffs():
            g_ = gathered
            if args.shard in ("rows", "peers"):
                return sharded.run(g_["x"], g_["y"], g_["w"], g_["K"], g_["area"])
            return sharded.run(g_["x"], g_["y"], g_["w"], g_["K"])
        out_bytes = plan.out.numel() * plan.out.element_size()
    else:
        plan = fcfs.CoeffsPlan(K, wl.T, wl.M, wl.N, wl.r2, layout, prec, device=dev, route=args.route)
        area_h = int(vp.area[0].item())

        def coeffs():
            return plan.run(vp.x[:K], vp.y[:K], vp.w[:K], area_h)
        out_bytes = plan.out.numel() * plan.out.element_size()
    graph_plan = None
    if (small is None and wl.B == 1 and world == 1 and args.input == "rects" and args.config != "layout"
            and not args.no_graph and args.route != "gemm"
            and fcfs.coeffs_route(K, wl.T, wl.M, wl.N, wl.r2, layout, prec, route=args.route) == 1):
        # one clip on the lattice-FFT route: the whole step (a1-a5) without a host sync, captured once in a
        # CUDA graph and replayed; the host-synchronising CoeffsPlan above stays for the stage timing
        graph_plan = fcfs.AsyncClipPlan(wl.R, wl.T, wl.M, wl.N, wl.r2, layout, prec, G=G, max_group=mg, device=dev)
        graph_plan.run(rects, gp)
        torch.cuda.synchronize()
        assert graph_plan.check() == K
        g_stream = torch.cuda.Stream(dev)
        graph = torch.cuda.CUDAGraph()
        lc0 = fcfs.kernel_launches()
        with torch.cuda.graph(graph, stream=g_stream):
            graph_plan.run(rects, gp, stream=g_stream)
        graph_launches = fcfs.kernel_launches() - lc0   # this library's kernels in one replay
        sync_coeffs, extract_sync = coeffs, extract

        def extract():
            return K

        def coeffs():
            graph.replay()
            return graph_plan.out
    def run_e2e():
        """The end-to-end measurement (below); returns the e2e dict or None."""
        # ---------------- end-to-end through the public API with host buffers
        # Batched clips: the step is cut into sub-batches whose H2D copy (rects, pinned), compute
        # (fcfs_vertices_from_rects + fcfs_coeffs_batched on a compute stream) and D2H copy (the
        # coefficients, into pinned memory) run on three streams, so the copies of one sub-batch overlap
        # the compute of the next.  Every byte of every step's input and output still crosses PCIe inside
        # the timed region (start / end events bracket all three streams).  One clip: sequential.
        e2e = None
        if not args.no_e2e and args.input == "rects":
            e2e_steps = max(3, args.steps)
            h2d_bytes = int(rects_h.numel() * 4)
            if wl.B > 1 and wl.B % args.e2e_split == 0 and wl.group_ptr is None and args.config != "layout":
                S = args.e2e_split
                bs = wl.B // S
                r_per = wl.clip_ptr[bs] - wl.clip_ptr[0]        # rects per sub-batch (equal clip sizes, c3)
                subs = []
                for i in range(S):
                    r0 = int(wl.clip_ptr[i * bs]); r1 = int(wl.clip_ptr[(i + 1) * bs])
                    cps = torch.from_numpy(wl.clip_ptr[i * bs:(i + 1) * bs + 1] - r0).to(dev)
                    vps = fcfs.VerticesPlan(r1 - r0, wl.T, r1 - r0, bs, 1, grouped=False, device=dev)
                    Ki = vps.run(rects[r0:r1].contiguous(), None, cps)
                    kmi = int(np.diff(vps.corner_ptr.cpu().numpy()).max())
                    pls = fcfs.BatchedPlan(bs, Ki, kmi, wl.T, wl.M, wl.N, wl.r2, layout, prec, device=dev,
                                           form=args.form, sorted_y=True)
                    subs.append({"r0": r0, "r1": r1, "cp": cps, "vp": vps, "plan": pls,
                                 "dev": torch.empty((r1 - r0, 4), dtype=torch.int32, device=dev),
                                 "out_h": torch.empty(pls.out.numel(), dtype=pls.out.dtype).pin_memory()})
                # one stream and one host thread per sub-batch: fcfs_vertices_from_rects synchronises its own
                # stream once (it returns K), so each sub-batch's pipeline (H2D -> extraction -> coefficients
                # -> D2H) is driven by its own thread and only blocks that thread; the copy engines and the
                # SMs overlap the sub-batches
                import concurrent.futures
                streams = [torch.cuda.Stream(dev) for _ in range(S)]
                pool = concurrent.futures.ThreadPoolExecutor(max_workers=S)

                def pipeline(i, ev0, steps):
                    # this sub-batch's work for every timed step, in order on its own stream
                    sb, st = subs[i], streams[i]
                    torch.cuda.set_device(dev)
                    st.wait_event(ev0)
                    with torch.cuda.stream(st):
                        for _ in range(steps):
                            sb["dev"].copy_(rects_h[sb["r0"]:sb["r1"]], non_blocking=True)
                            kk = sb["vp"].run(sb["dev"], None, sb["cp"], stream=st)
                            o = sb["plan"].run(sb["vp"].corner_ptr, sb["vp"].x[:kk], sb["vp"].y[:kk], sb["vp"].w[:kk],
                                               sb["vp"].area, stream=st)
                            sb["out_h"].copy_(o.reshape(-1), non_blocking=True)
                        done = torch.cuda.Event()
                        done.record(st)
                    return done
                torch.cuda.synchronize()
                if world > 1:
                    dist.barrier()
                ea, eb = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                main = torch.cuda.current_stream(dev)
                ea.record(main)
                for d in [f.result() for f in [pool.submit(pipeline, i, ea, e2e_steps) for i in range(S)]]:
                    main.wait_event(d)
                eb.record(main)
                torch.cuda.synchronize()
                pool.shutdown()
                e2e_note = (f"{S} sub-batches of {bs} clips, one stream + host thread each running H2D, extraction, "
                            f"coefficients, D2H for every step in order (a streaming pipeline: sub-batches and steps "
                            f"overlap; every step's bytes cross PCIe inside the events)")
            else:
                out_h = torch.empty(plan.out.numel(), dtype=plan.out.dtype).pin_memory()
                torch.cuda.synchronize()
                if world > 1:
                    dist.barrier()
                ea, eb = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                ea.record()
                for _ in range(e2e_steps):
                    rects.copy_(rects_h, non_blocking=True)
                    extract()
                    o = coeffs()
                    out_h.copy_(o.reshape(-1), non_blocking=True)
                eb.record()
                torch.cuda.synchronize()
                e2e_note = "sequential: H2D, step, D2H"
            te = torch.tensor([ea.elapsed_time(eb)], dtype=torch.float64, device=dev)
            if world > 1:
                dist.all_reduce(te, op=dist.ReduceOp.MAX)
            e2e = {"value": terms * world * e2e_steps / (float(te.item()) / 1e3) / 1e9, "unit": "Gterm/s",
                   "h2d_bytes_per_step": h2d_bytes, "d2h_bytes_per_step": int(out_bytes), "steps": e2e_steps,
                   "pipeline": e2e_note}


        return e2e

    e2e_early = None
    terms = float(W) * float(K)                     # per rank per step (batched clips: not sharded)
    if (graph_plan is None and small is None and wl.B > 1 and wl.group_ptr is None and args.input == "rects"
            and args.config != "layout" and not args.no_graph and plan.form == 3 and vp is not None):
        # the end-to-end run goes first: measured after the capture it read ~10% lower (18.5K vs 20.6K
        # Gterm/s), an effect of the captured graph on the later host-driven pipeline that we did not isolate
        e2e_early = run_e2e()
        # batched clips on the lattice-row form: sync-free extraction (fcfs_vertices_from_clips_async, the
        # per-clip bucket kernel with the rects-per-clip bound given) + fcfs_coeffs_batched (sorted_y: no sync)
        # captured once as a CUDA graph and replayed; the host-synchronising calls above stay for the stage
        # timing.  K_total / K_max of the plan are the workload's (fixed rects); the kernels read corner_ptr.
        max_clip_rects = int(np.diff(wl.clip_ptr).max())
        vp.run_clips_async(rects, cp, max_clip_rects)
        torch.cuda.synchronize()
        assert vp.check_async() == K
        g_stream = torch.cuda.Stream(dev)
        graph = torch.cuda.CUDAGraph()
        lc0 = fcfs.kernel_launches()
        with torch.cuda.graph(graph, stream=g_stream):
            vp.run_clips_async(rects, cp, max_clip_rects, stream=g_stream)
            plan.run(vp.corner_ptr, vp.x[:K], vp.y[:K], vp.w[:K], vp.area, stream=g_stream)
        graph_launches = fcfs.kernel_launches() - lc0
        graph_plan = plan
        sync_coeffs, extract_sync = coeffs, extract

        def extract():
            return K

        def coeffs():
            graph.replay()
            return plan.out
    terms = float(W) * float(K)                     # per rank per step
    single_sharded = wl.B == 1 and world > 1
    if single_sharded:
        terms /= world                              # one clip split over the ranks: value = total terms / time
    flush = torch.empty(512 * 1024 * 1024, dtype=torch.uint8, device=dev)

    def step():
        extract()
        return coeffs()

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()

    # ---------------- timed region (device-timed: events per step, L2 flushed between steps)
    fcfs.profile_enable(True)
    fcfs.profile_read()
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    launches0 = fcfs.kernel_launches()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    with ClockSampler(local) as clk:
        for i in range(args.steps):
            evs[i][0].record()
            step()
            evs[i][1].record()
            flush.fill_(i & 0xff)
        torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    launches = fcfs.kernel_launches() - launches0 + graph_launches * args.steps
    stages = fcfs.profile_read()
    fcfs.profile_enable(False)
    per_rank = None
    if world > 1:
        allst = [None] * world
        dist.all_gather_object(allst, {k: round(v[0] / args.steps, 4) for k, v in stages.items()})
        per_rank = allst
    step_ms = [a.elapsed_time(b) for a, b in evs]
    total_ms = sum(step_ms)
    t = torch.tensor([total_ms], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    total_ms = float(t.item())
    ms_per_step = total_ms / args.steps
    value = terms * world * args.steps / (total_ms / 1e3) / 1e9

    # ---------------- roofline of the dominant kernel (the a3 contraction)
    peaks, src = load_peaks()
    if graph_plan is not None:
        # stage times of the same work through the host-synchronising calls (outside the timed region)
        fcfs.profile_enable(True)
        fcfs.profile_read()
        for _ in range(args.steps):
            extract_sync()
            sync_coeffs()
        torch.cuda.synchronize()
        stages = fcfs.profile_read()
        fcfs.profile_enable(False)
    c_ms, c_n = stages["contract"]
    c_ms_launch = c_ms / max(c_n, 1)
    fft_route = (small is None and wl.B == 1 and world == 1 and
                 fcfs.coeffs_route(K, wl.T, wl.M, wl.N, wl.r2, layout, prec, route=args.route) == 1)
    if small is not None:
        # one kernel per step (a graph of one launch): its time is the step's; algorithmic work = the
        # direct sums over the half window, one complex MAC (8 flop) per (output, corner)
        c_ms_launch = ms_per_step
        alg_flops = 8.0 * (W / 2.0) * K
        achieved = alg_flops / (c_ms_launch / 1e3) / 1e12
        clocks = clk.summary()
        try:
            peak = json.load(open(os.path.join(ROOT, "profiles", "fp64_peak.json")))["dfma_tflops"]
            peak_note = "FP64 CUDA-core DFMA measured by tools/fp64_peak.cu (profiles/fp64_peak.json)"
        except Exception:
            mhz = peaks.get("sm_max_mhz", 1965.0)
            peak = 148 * 64 * 2 * mhz * 1e6 / 1e12
            peak_note = f"FP64 DFMA derived: 148 SM x 64 FMA/clk x 2 x {mhz:.0f} MHz"
        peak_note += "; latency-bound (one launch per step, the whole clip in every CTA's shared memory)"
        bound = "alu"
        k_inner = "canonical corners (direct sums, fcfs_small_clip)"
        Kc = np.array([float(K)])
    elif fft_route:
        # lattice-FFT route (NEXT-2, FP64 or FP32 CUDA cores): algorithmic work of the contract stage =
        # G rows (one complex rotation + real-weighted complex MAC per corner and row: 10 flop) +
        # the T1 length-T2 FFTs per row (5 T2 log2 T2) + the outer twiddled sum (8 flop per n and y1)
        T2 = 64
        while T2 < 2 * wl.N + 1:
            T2 *= 2
        T1 = wl.T // T2
        rows = wl.M + 1
        alg_flops = (10.0 * K * wl.M + rows * T1 * (5.0 * T2 * math.log2(T2) + 8.0 * (2 * wl.N + 1)))
        achieved = alg_flops / (c_ms_launch / 1e3) / 1e12
        clocks = clk.summary()
        if prec == "fp64":
            try:
                peak = json.load(open(os.path.join(ROOT, "profiles", "fp64_peak.json")))["dfma_tflops"]
                peak_note = ("FP64 CUDA-core DFMA measured by tools/fp64_peak.cu on this pool "
                             f"(profiles/fp64_peak.json); the stage = k_fr_rows + k_fr_fft2 + small kernels, "
                             f"T2={T2}, T1={T1}")
            except Exception:
                mhz = peaks.get("sm_max_mhz", 1965.0)
                peak = 148 * 64 * 2 * mhz * 1e6 / 1e12
                peak_note = f"FP64 DFMA derived: 148 SM x 64 FMA/clk x 2 x {mhz:.0f} MHz; T2={T2}, T1={T1}"
        else:
            mhz = peaks.get("sm_max_mhz", 1965.0)
            peak = 148 * 128 * 2 * mhz * 1e6 / 1e12
            peak_note = (f"FP32 CUDA-core FFMA, derived: 148 SM x 128 lanes x 2 flop x {mhz:.0f} MHz (the FP32 "
                         f"route of the split precisions); stage = k_fr_rows + k_fr_fft2 + small kernels, "
                         f"T2={T2}, T1={T1}")
        bound = "alu"
        k_inner = "lattice-FFT route"
        Kc = np.array([float(K)])
    else:
        # inner dimension of the contraction: corners (batched tcgen05 kernels) or row buckets (FP64, and
        # split-TF32 on one clip: Step 4 row structure, fcfs_row_buckets with the cap fcfs_coeffs uses)
        if prec == "fp64" or wl.B == 1:
            ysrc = vp.y if vp is not None else gathered["y"]
            rb = fcfs.row_buckets(ysrc[:K], vp.corner_ptr if wl.B > 1 else None, 32)
            Kc = np.diff(rb["clip_bptr"].cpu().numpy()).astype(np.float64)
            k_inner = "row buckets"
        elif getattr(plan, "form", 0) == fcfs.FORM_LATTICE:
            # lattice-row form: the tensor GEMM contracts over the T+1 lattice rows of every clip
            Kc = np.full(wl.B, float(wl.T + 1))
            k_inner = "lattice rows (T+1 per clip)"
        elif getattr(plan, "form", 0) == fcfs.FORM_EDGE:
            Kc = edge_counts(vp, K, cptr_h)
            k_inner = "edges (K/2-term form)"
        else:
            Kc = np.diff(cptr_h).astype(np.float64)
            k_inner = "corners"
        alg_flops = float(np.sum(8.0 * wl.M * wl.N * Kc))      # real quadrant GEMM 2M x 2N x K_inner, 2 flop/MAC
        achieved = alg_flops / (c_ms_launch / 1e3) / 1e12
        clocks = clk.summary()
        if prec == "tf32x3":
            tf32 = peaks["bf16_tflops"] * (1.1 / 2.25)
            peak = tf32 / 3.0
            peak_note = (f"TF32 dense = {src} bf16 {peaks['bf16_tflops']} x (1.1/2.25 nominal ratio) = {tf32:.1f} "
                         f"TF/s, / 3 (split-TF32: 3 TF32 MMAs per FP32-accurate product)")
            bound = "tensor"
        elif prec == "f16x3":
            peak = peaks["bf16_tflops"] / 3.0
            peak_note = (f"FP16 dense = {src} bf16 {peaks['bf16_tflops']} TF/s (same nominal rate), / 3 "
                         f"(split-FP16: 3 FP16 MMAs per FP32-accurate product)")
            bound = "tensor"
        else:
            try:
                peak = json.load(open(os.path.join(ROOT, "profiles", "fp64_peak.json")))["dmma_m16n8k16_tflops"]
                peak_note = "FP64 tensor (DMMA m16n8k16) measured by tools/fp64_peak.cu on this pool (profiles/fp64_peak.json)"
            except Exception:
                mhz = peaks.get("sm_max_mhz", 1965.0)
                peak = 148 * 64 * 2 * mhz * 1e6 / 1e12
                peak_note = f"FP64: 148 SM x 64 FMA/clk x 2 x {mhz:.0f} MHz (derived)"
            bound = "tensor"
    roof = {"bound": bound, "achieved": round(achieved, 3), "peak": round(peak, 3), "unit": "TFLOP/s",
            "frac": round(achieved / peak, 4), "traffic": traffic_for(args.config, prec, "fft" if fft_route else
                                   ("corners" if (prec == "tf32x3" and wl.B > 1 and k_inner == "corners") else
                                    "edges" if (prec == "tf32x3" and wl.B > 1 and k_inner.startswith("edges")) else "")),
            "step": ("sync-free a1-a5 (fcfs_vertices_from_rects_async + fcfs_coeffs_async) replayed as a CUDA graph; "
                     "stage times from the host-synchronising calls" if graph_plan is not None else None),
            "kernel": ("k_small_clip (a1-a5 in one launch, CUDA graph replay)" if small is not None else
                       f"contract stage (lattice-FFT route, {'FP64' if prec == 'fp64' else 'FP32'}: k_fr_rows + k_fr_fft2)"
                       if fft_route else ("contract stage (lattice-row form: k_lat_btab + k_lat_cptr + k_lattice)"
                                          if getattr(plan, "form", 0) == fcfs.FORM_LATTICE else "k_gemm_" + prec)),
            "k_inner": f"{k_inner}: {int(Kc.sum())}",
            "alg_flops_per_launch": alg_flops,
            "kernel_ms_per_launch": round(c_ms_launch, 4), "peak_source": peak_note,
            "stage_ms_per_step": {k: round(v[0] / args.steps, 4) for k, v in stages.items()}}

    e2e = e2e_early if e2e_early is not None else run_e2e()

    if rank == 0:
        line = {"metric": "fourier_coeff_vertex_terms_per_sec", "value": round(value, 3), "unit": "Gterm/s",
                "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms_per_step, 4),
                "higher_is_better": True, "scaling": "strong" if single_sharded else "weak", "vs_baseline": None,
                "dtype": ("f64" if (prec == "fp64" or small is not None) else
                          "f32 (lattice-FFT route on FP32 CUDA cores, FP64 outer sums; the split-precision contract)"
                          if fft_route else
                          "tf32x3 (split-TF32, FP32-accurate; FP64 flush)" if prec == "tf32x3" else
                          "f16x3 (split-FP16, FP32-accurate; FP64 flush)"),
                "data": "synthetic", "config": config_dict(args, wl, prec, world),
                "K_per_gpu": int(K), "terms_per_step_per_gpu": terms,
                "roofline": roof, "clocks": clocks, "gpu_launches": int(launches),
                "e2e": e2e}
        if per_rank is not None:
            line["per_rank_stage_ms_per_step"] = per_rank
        if world == 1 and not args.no_cpu_baseline:
            line["cpu_baseline"] = cpu_baseline(wl, args.cpu_seconds, prec)
        if (world == 1 and args.config == "c3" and not args.no_extra and args.prec in (None, "tf32x3")
                and args.input == "rects"):
            line["extra"] = run_extras(args)
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
