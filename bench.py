#!/usr/bin/env python
"""Benchmark: simplex iterations/s on BASELINE.json's headline config.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config c3] [--impl ours|reference]
                    [--e2e-max-iter N] [--no-cpu-baseline] [--no-reinversion] [--transport p2p|nccl]

A "step" is one pivot of the dense revised simplex (one pass of the hot path:
pivot row, pricing, fused update + FTRAN + ratio test) on a synthetic LP from
the reference's own generator (seed 1), resident in HBM. W warm-up pivots run
first (untimed), then exactly K pivots are timed with CUDA events on the
solver's stream (`value`), and through the public API with the host clock
(`e2e`, the same window). The working set (A: 1.0 GB, B^-1: 0.5 GB at m=8000)
is far larger than the 126 MB L2, so no flush is needed between pivots.

The line also carries the time to the final status (parity mode, the
reference's own outcome) and, opt-in, with periodic reinversion; the roofline
of the dominant kernel; and the unmodified reference CPU solver timed on the
same LP and pivot window (`cpu_baseline`).

Prints ONE JSON line (rank 0). `--impl reference` times the reference's own
CPU implementation (oracle/_ref, i.e. lps::two_phase_solve compiled from the
unmodified reference sources) on the LP the reference itself generates (same
SHA-256, printed in `config`), over the same pivot window, with all host cores.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

CONFIGS = {
    # BASELINE.json configs[0..4]
    "c1": dict(rows=256, cols=512, form=1, seed=1, cpu_pivots=824, w1_steps=800, reinv_every=500,
               label="C1 random dense LP m=256 n=512 (<= rows, maximize; slack start), seed 1"),
    "c2": dict(rows=2000, cols=4000, form=0, seed=1, cpu_pivots=300, w1_steps=100, reinv_every=2000,
               label="C2 random dense LP m=2000 n=4000 (generator verbatim, equality rows), seed 1"),
    "c3": dict(rows=8000, cols=16000, form=0, seed=1, cpu_pivots=60, w1_steps=20, reinv_every=50000,
               label="C3 random dense LP m=8000 n=16000 (generator verbatim, equality rows), seed 1"),
    "c4": dict(rows=4000, cols=8000, form=2, seed=1, cpu_pivots=1, ref_max_steps=1,
               label="C4 degenerate LP m=4000 n=8000 (<= rows, maximize, half the rows a_i - a_i+1 "
                     "with b_i = 0), seed 1"),
    "c5": dict(rows=24000, cols=48000, form=0, seed=1, cpu_pivots=5,
               label="C5 random dense LP m=24000 n=48000 (generator verbatim), seed 1"),
}
def _metric():
    try:
        with open(os.path.join(ROOT, "BASELINE.json")) as f:
            return json.load(f)["metric"]
    except Exception:
        return "simplex iterations/sec & time-to-optimal, dense LP m=8000 @1/2/4/8 B200"


METRIC = _metric()
NOMINAL_HBM_GBS = 8000.0
NCU_NAMES = {"price": "k_price", "update_ftran": "k_update", "pivot": "k_pivot", "ratio": "k_ratio"}


def _ncu_traffic(kernel: str):
    """DRAM bytes (read + write) per launch of `kernel` from the newest committed
    `ncu --set full` summary under profiles/ (tools/ncu_summary.py), or None."""
    import glob
    best = None
    # a checkout gives every file the same mtime: the latest round's summary
    # (r02 > r01) wins, then a *_final_* one
    def rank(p):
        b = os.path.basename(p)
        return (b[:3], "_final_" in b, os.path.getmtime(p))
    for p in sorted(glob.glob(os.path.join(ROOT, "profiles", "*_ncu_summary.json")), key=rank):
        try:
            with open(p) as f:
                cap = json.load(f).get("captures", {}).get(kernel)
            if cap and cap.get("traffic_bytes"):
                best = (cap["traffic_bytes"], os.path.basename(p))
        except Exception:
            pass
    return best


def _sm_max_mhz() -> float:
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return float(json.load(f)["sm_max_mhz"])
    except Exception:
        return 1965.0


def _peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int, interval: float = 0.2):
        self.device = device
        self.interval = interval
        self.rows = []
        self._stop = threading.Event()
        self._t = None

    def __enter__(self):
        def run():
            while not self._stop.is_set():
                try:
                    out = subprocess.run(["nvidia-smi", "-i", str(self.device),
                                          f"--query-gpu={self.Q}", "--format=csv,noheader,nounits"],
                                         capture_output=True, text=True, timeout=5).stdout
                    for line in out.strip().splitlines():
                        self.rows.append([v.strip() for v in line.split(",")])
                except Exception:
                    pass
                self._stop.wait(self.interval)
        self._t = threading.Thread(target=run, daemon=True)
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self._t:
            self._t.join(timeout=6)

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"], "samples": 0}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[k] for r in self.rows for k in range(4)
                          if len(r) > 3 + k and r[3 + k].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "samples": len(self.rows)}


def make_lp(cfg, pinned=False):
    import paper_1803_04378_b200 as P
    return P.generate(P.GenSpec(cfg["rows"], cfg["cols"], P.SparsityClass.dense, cfg["seed"],
                                P.Form(cfg["form"])), pinned=pinned)


def lp_digest(A, b, c, col_kind) -> str:
    """SHA-256 of the standard-form arrays: both arms print it in `config`, so
    equal configs mean bit-identical inputs (the reference arm draws its LP with
    the reference's own generate + canonicalize, ours with lpsg_generate)."""
    import hashlib

    import numpy as np
    h = hashlib.sha256()
    for a in (A, b, c, col_kind):
        h.update(memoryview(np.ascontiguousarray(a)).cast("B"))
    return h.hexdigest()


def bench_config(cfg, m, n_total, digest, W, K):
    """The `config` object, identical in both arms for the same workload."""
    return {"workload": cfg["label"], "m": m, "n_total": n_total, "lp_sha256": digest,
            "pivots_timed": [W, W + K],
            "l2": "working set > L2 (A 8*m*n_total B, B^-1 8*m^2 B); no flush needed"}


def cpu_reference_window(lp, W, K, workers):
    """The reference CPU solver (oracle/_ref: lps::two_phase_solve compiled from
    the unmodified sources; the C port if that library is absent) on the pivot
    window [W, W+K) of `lp`, timed by per-pivot observer timestamps inside
    solve() (solver.cpp:264-275, 332). Returns (it/s, pivots, seconds, kind)."""
    from oracle.oracle import LP, Port, Ref, make_config
    olp = LP(lp.m, lp.n_total, lp.A, lp.b, lp.c, lp.col_kind)
    try:
        ref = Ref()
    except Exception:  # noqa: BLE001
        port = Port()
        out = port.solve(olp, make_config(max_iter=W + K), trace_cap=0)
        n = out.iterations_phase1 + out.iterations_phase2
        return (n / out.total_seconds if out.total_seconds > 0 else None), n, out.total_seconds, "port"
    secs, done, _ = ref.solve_window(olp, make_config(workers=workers), W, K)
    return (done / secs if secs > 0 else None), done, secs, "reference"


def reference_best(lp, W, K, cfg):
    """cpu_reference_window with workers = nproc and (bounded by the config's
    w1_steps) workers = 1. The reference threads only its pricing loop
    (solver.cpp:99-121), so one worker can be the faster setting at small m:
    the faster of the two is reported when both cover the same window.
    Returns (it/s, pivots, seconds, kind, workers used, workers-1 dict|None)."""
    cores = os.cpu_count() or 1
    val, done, secs, kind = cpu_reference_window(lp, W, K, cores)
    used = cores if kind == "reference" else 1
    w1 = None
    if kind == "reference" and cfg.get("w1_steps", 0):
        k1 = min(K, cfg["w1_steps"])
        v1, d1, s1, _ = cpu_reference_window(lp, W, k1, 1)
        w1 = {"value": v1, "pivots": [W, W + d1], "seconds": s1}
        if d1 == done and v1 and val and v1 > val:
            val, secs, used = v1, s1, 1
    return val, done, secs, kind, used, w1


def reference_lp(cfg):
    """The LP as the reference itself builds it: lps::generate + the input form
    + lps::canonicalize (oracle/ref_shim.cpp ref_lp_generate). No lpsg code."""
    from oracle.oracle import Port, Ref
    try:
        return Ref().generate(cfg["rows"], cfg["cols"], cfg["seed"], cfg["form"])
    except Exception:  # noqa: BLE001
        return Port().generate(cfg["rows"], cfg["cols"], cfg["seed"], cfg["form"])


def run_reference_arm(args, cfg):
    """`--impl reference`: the unmodified reference (oracle/_ref) on the same LP
    (digest in config), the same pivot window [W, W+K) and the same config
    object as our arm, with every host thread (cfg.workers = nproc); rank 0
    only. Never loads liblpsg."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    lp = reference_lp(cfg)
    digest = lp_digest(lp.A, lp.b, lp.c, lp.col_kind)
    W, K = args.warmup, args.steps
    cap = cfg.get("ref_max_steps")
    if cap is not None and W + K > cap:  # C4: ~200 s per tie pivot on the CPU
        W, K = 0, cap
    cores = os.cpu_count() or 1
    val, done, secs, kind, used, w1 = reference_best(lp, W, K, cfg)
    line = {
        "impl": "reference", "metric": METRIC, "value": val, "unit": "iterations/s",
        "n_gpus": args.gpus, "steps": done, "warmup": W,
        "ms_per_step": 1e3 * secs / max(1, done),
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (reference generator lps::generate, seed 1)",
        "config": bench_config(cfg, lp.m, lp.n_total, digest, W, done),
        "cpu_baseline": {"value": val, "unit": "iterations/s", "cores": used, "kind": kind,
                         "sample": f"pivots [{W}, {W + done}) of {cfg['label']}: lps::two_phase_solve "
                                   f"(oracle/_ref, unmodified sources), best of workers = {cores} "
                                   f"and workers = 1 (here {used}), per-pivot observer timestamps "
                                   f"({secs:.2f} s)"},
        "e2e": {"value": val, "unit": "iterations/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    if w1 is not None:
        line["cpu_baseline"]["workers_1"] = w1
    print(json.dumps(line), flush=True)


# ---- multi-GPU control plane (torchrun: one process per GPU). The solver's
# data path is NCCL inside liblpsg; torch.distributed (gloo) only hands out the
# NCCL unique id and takes the max of the per-rank device times.
def dist_ctx():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", str(rank)))
    if os.environ.get("LPSG_BENCH_SAME_DEVICE"):
        local = 0  # testing the multi-process path on a one-GPU box (time-sliced, not a bench number)
    if world > 1:
        import torch.distributed as dist
        if not dist.is_initialized():
            dist.init_process_group("gloo")
    return world, rank, local


def share_nccl_id(world: int, rank: int) -> bytes:
    """A fresh NCCL unique id from rank 0, identical on every rank."""
    import paper_1803_04378_b200 as P
    import torch.distributed as dist
    obj = [P.nccl_unique_id() if rank == 0 else None]
    dist.broadcast_object_list(obj, src=0)
    return obj[0]


def max_over_ranks(v: float, world: int) -> float:
    if world == 1:
        return float(v)
    import torch
    import torch.distributed as dist
    t = torch.tensor([float(v)], dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def barrier(world: int) -> None:
    if world > 1:
        import torch.distributed as dist
        dist.barrier()


_PEER = None


def peer_heap(world: int, rank: int, local: int):
    """The P2P transport's symmetric heap, connected once per process: every
    rank all-gathers the 64-byte CUDA IPC handles over gloo."""
    global _PEER
    if _PEER is None:
        import paper_1803_04378_b200 as P
        import torch.distributed as dist
        # every step is agreed by all ranks, so a failure on any rank raises on
        # all of them together and they fall back to NCCL in step (main())
        h, err = None, ""
        try:
            h = P.PeerHeap(rank, world, device=local)
        except Exception as e:  # noqa: BLE001
            err = f"rank {rank}: {e}"
        handles = [None] * world
        dist.all_gather_object(handles, h.handle if h is not None else None)
        if h is not None and all(x is not None for x in handles):
            try:
                h.connect(handles)
            except Exception as e:  # noqa: BLE001
                err = f"rank {rank}: {e}"
        errs = [None] * world
        dist.all_gather_object(errs, err)
        bad = [e for e in errs if e] or ([] if all(x is not None for x in handles)
                                          else ["a rank has no peer heap"])
        if bad:
            raise RuntimeError("P2P heap unavailable: " + "; ".join(bad))
        _PEER = h
    return _PEER


def solver_config(P, args, world, rank, local, **kw):
    extra = {}
    if world > 1:
        if args.transport == "p2p":
            extra = dict(peer=peer_heap(world, rank, local))
        else:
            extra = dict(world_size=world, rank=rank, nccl_id=share_nccl_id(world, rank))
    return P.SolverConfig(device=local if world > 1 else 0, batch=args.batch, **extra, **kw)


def run_ours(args, cfg):
    import paper_1803_04378_b200 as P
    world, rank, local = dist_ctx()
    device = local if world > 1 else 0
    lp = make_lp(cfg, pinned=True)  # every lpsg_create uploads from page-locked memory
    W, K = args.warmup, args.steps

    # ---- device-resident timing: W warm-up pivots, then K timed pivots (the
    # value; no per-kernel events), then K more pivots with per-kernel CUDA
    # events on the solver stream (the roofline). The time is the max over ranks
    # of each rank's CUDA-event span on its solver stream.
    s = P.SimplexSolver(lp, solver_config(P, args, world, rank, local, max_iter=W))
    s.solve()
    c0 = s.counters()
    x0 = s.comm_stats()
    s.set_max_iter(W + K)
    barrier(world)
    with ClockSampler(device) as clk:
        # the same window through the public API, by the host clock: lpsg_solve
        # (per-batch control-block H2D, pivot-log D2H) + lpsg_get_x (x D2H)
        t0 = time.perf_counter()
        rep = s.solve()
        t1 = time.perf_counter()
    barrier(world)
    dev_ms = max_over_ranks(s.device_ms(), world)
    wall_window = max_over_ranks(t1 - t0, world)
    c1 = s.counters()
    x1 = s.comm_stats()
    done = rep.iterations - W
    value = done / (dev_ms / 1e3)
    e2e = {"value": done / wall_window, "unit": "iterations/s",
           "h2d_bytes_per_step": (c1["h2d_bytes"] - c0["h2d_bytes"]) / max(1, done),
           "d2h_bytes_per_step": (c1["d2h_bytes"] - c0["d2h_bytes"] + 8 * lp.n_total) / max(1, done),
           "includes": f"host clock around lpsg_solve + lpsg_get_x over pivots [{W}, {W + done}) "
                       "(the window `value` times on the device): control-block H2D and "
                       "pivot-log D2H per batch, host decisions, x D2H; the LP was uploaded "
                       "from pinned host memory by lpsg_create before the window, as the "
                       "reference's constructor runs before its solve() clock "
                       "(solver.cpp:332); max over ranks"}
    stats = {}
    prof_range = None
    done_p = 0
    if not args.no_profile:
        s.set_max_iter(W + 2 * K)
        s.profile(True)
        rep_p = s.solve()
        stats = s.profile_stats()
        prof_range = [W + done, rep_p.iterations]
        done_p = rep_p.iterations - W - done
    la_stats = s.lookahead_stats()
    s.close()

    # ---- roofline of the dominant kernel (per GPU) and of the whole pivot
    peak, peak_kind = _peaks()
    kern = {}
    for name, st in stats.items():
        if st["launches"] and st["ms"] > 0:
            kern[name] = dict(launches=st["launches"], ms_total=round(st["ms"], 4),
                              us_per_launch=round(1e3 * st["ms"] / st["launches"], 3),
                              share=None)
            if name.startswith("lookahead"):  # compute-bound: "bytes" are fp64 flops
                kern[name]["tflops"] = round(st["bytes"] / (st["ms"] / 1e3) / 1e12, 3)
            else:
                kern[name]["gbs"] = (round(st["bytes"] / (st["ms"] / 1e3) / 1e9, 1)
                                     if st["bytes"] else None)
    tot = sum(v["ms_total"] for v in kern.values()) or 1.0
    for v in kern.values():
        v["share"] = round(v["ms_total"] / tot, 4)
    roofline = None
    traffic = None
    if kern:
        hbm = {k: v for k, v in kern.items() if v.get("gbs")}
        dom = max(hbm, key=lambda k: hbm[k]["ms_total"])
        ach = kern[dom]["gbs"]
        # algorithmic bytes of one pivot on this rank; the whole job moves world x that
        pivot_bytes = sum(stats[k]["bytes"] for k in stats if not k.startswith("lookahead")) / max(1, done_p)
        job_gbs = pivot_bytes * world * value / 1e9
        roofline = {"bound": "hbm", "kernel": dom, "achieved": ach, "peak": peak, "unit": "GB/s",
                    "frac": round(ach / peak, 4), "traffic": None, "peak_source": peak_kind,
                    "frac_nominal": round(ach / NOMINAL_HBM_GBS, 4),
                    "peak_note": "peak = MEASURED_PEAKS.json hbm_gbs, a device-to-device copy "
                                 "(read + write); read-only streams such as k_price can exceed "
                                 f"it; frac_nominal is against the {NOMINAL_HBM_GBS:.0f} GB/s "
                                 "HBM3e nominal",
                    "per_pivot": {"algorithmic_bytes_per_gpu": pivot_bytes,
                                  "achieved_gbs_per_gpu": round(job_gbs / world, 1),
                                  "frac": round(job_gbs / world / peak, 4),
                                  "frac_nominal": round(job_gbs / world / NOMINAL_HBM_GBS, 4)},
                    "kernels": kern, "instrumented_pivots": prof_range,
                    "note": "per-kernel CUDA events on the solver stream over a second window of "
                            "K pivots (rank 0); the headline value is the un-instrumented window"}
        # the other floor of a pivot: pricing and FTRAN are each one sequential
        # chain of m fp64 adds per output (8-cycle DADD latency, measured), plus
        # three kernel boundaries. Small m (C1, C2) sits on this floor, not on HBM.
        clk_ghz = _sm_max_mhz() / 1e3
        chain_us = 2 * (lp.m + 1) * 8 / clk_ghz / 1e3
        hbm_us = pivot_bytes / (peak * 1e9) * 1e6
        roofline["latency_floor"] = {
            "chain_us_per_pivot": round(chain_us, 2), "hbm_us_per_pivot": round(hbm_us, 2),
            "measured_us_per_pivot": round(1e6 / value, 2) if value else None,
            "regime": "hbm" if hbm_us >= chain_us else "chain/latency",
            "note": "chain = 2 sequential dots of m+1 DADDs at 8 cycles (pricing, FTRAN); the "
                    "pivot cannot beat max(chain, hbm)"}
        la = {k: v for k, v in kern.items() if "tflops" in v}
        la_ms = sum(v["ms_total"] for v in la.values())
        if la and la_ms > sum(v["ms_total"] for v in hbm.values()):
            # tie pivots dominate (C4): the batched lookahead GEMMs are fp64
            # SIMT compute-bound (DMUL + DADD per multiply-add, no FMA, no tensor
            # cores: either would change the bits), so the roofline is the fp64 pipe
            ldom = max(la, key=lambda k: la[k]["ms_total"])
            fpk = P.fp64_peak(device)
            src = ("measured in this run: lpsg_fp64_peak (independent DMUL/DADD chains on all SMs, "
                   "1 flop per instruction)")
            if ldom == "lookahead_price" and la_stats["price_bounded"]:
                # the bounded pricing's screen runs on the fp64 tensor cores (DMMA
                # m8n8k4): 37.1 TFLOP/s measured, 2 x the DMUL/DADD instruction rate
                # (tools/microbench/dmma_rate.cu)
                fpk *= 2
                src += ("; x 2 for the bounded pricing's DMMA screen (fp64 tensor cores, "
                        "tools/microbench/dmma_rate.cu: 37.1 TFLOP/s)")
            roofline = {"bound": "fp64", "kernel": ldom, "achieved": la[ldom]["tflops"],
                        "peak": round(fpk, 2), "unit": "TFLOP/s",
                        "frac": round(la[ldom]["tflops"] / fpk, 4), "traffic": None,
                        "peak_source": src,
                        "lookahead_share_of_profiled_time": round(la_ms / tot, 4),
                        "lookahead_tflops_all": round(sum(stats[k]["bytes"] for k in la) /
                                                      (la_ms / 1e3) / 1e12, 3),
                        "hbm_side": {"kernel": dom, "achieved_gbs": ach, "peak_gbs": peak,
                                     "frac": round(ach / peak, 4)},
                        "kernels": kern, "instrumented_pivots": prof_range,
                        "note": "fp64 flops of the batched lookahead: 2 per pricing term "
                                "(K x m x n_scan) and 4 per theta term (K x m x m: the updated "
                                "element T_ij - y_i X_kj, then its product into y'); per-kernel "
                                "CUDA events on the solver stream over a second window"}
        t = _ncu_traffic(NCU_NAMES.get(dom, dom)) if args.config == "c3" else None  # captures are of C3
        if t is not None and world == 1:
            traffic = t[0]
            roofline["traffic_source"] = f"profiles/{t[1]} (ncu --set full, one launch, DRAM read+write bytes)"
        if traffic is not None:
            roofline["traffic"] = traffic
    exchange = None
    if world > 1:
        calls = (x1["calls"] - x0["calls"]) / max(1, done)
        nbytes = (x1["bytes"] - x0["bytes"]) / max(1, done)
        ex = kern.get("exchange")
        oth = kern.get("other")  # k_price_final / k_ratio_final: the flag waits + merges
        exchange = {"transport": ("P2P: device-initiated NVLink stores + sequence flags (CUDA IPC heaps)"
                                  if args.transport == "p2p" else "NCCL (NVLink/NVSwitch)"),
                    "collectives_per_pivot": round(calls, 2),
                    "payload_bytes_per_pivot_per_rank": round(nbytes, 1),
                    "us_per_pivot": round(1e3 * ex["ms_total"] / max(1, done_p), 2) if ex else None,
                    "us_per_pivot_incl_merge_kernels": round(
                        1e3 * ((ex["ms_total"] if ex else 0.0) + (oth["ms_total"] if oth else 0.0)) /
                        max(1, done_p), 2),
                    "note": "per pivot: pivot-row broadcast from its owner (m+3 words), the (z, j) "
                            "and ratio-message exchanges (P2P: stored into the peers' mailboxes by the "
                            "producing kernels' last CTA, no collective launch; NCCL: all-gathers)"}

    # ---- time-to-optimal through the public API with host buffers:
    # lpsg_create uploads A from pinned host memory, solve() runs from the start
    # basis to its final status (or the --e2e-max-iter budget), x is read back.
    cfg2 = solver_config(P, args, world, rank, local, max_iter=args.e2e_max_iter)
    barrier(world)
    # (no nvidia-smi sampling here: each call stalls the host side of the
    # create/upload it overlaps, ~0.7 s over this region in a measured A/B)
    t0 = time.perf_counter()
    s2 = P.SimplexSolver(lp, cfg2)
    rep2 = s2.solve()
    x = rep2.x  # solve() already read x back (device -> host)
    t1 = time.perf_counter()
    cnt = s2.counters()
    tto_dev = max_over_ranks(s2.device_ms() / 1e3, world)
    s2.close()
    wall = max_over_ranks(t1 - t0, world)
    tto = {"status": rep2.status.name, "objective": rep2.objective,
           "iterations_phase1": rep2.iterations_phase1,
           "iterations_phase2": rep2.iterations_phase2,
           "seconds_e2e": wall, "seconds_solve": rep2.total_seconds,
           "seconds_device": tto_dev, "iterations_per_s_e2e": rep2.iterations / wall,
           "h2d_bytes": cnt["h2d_bytes"], "d2h_bytes": cnt["d2h_bytes"] + 8 * len(x),
           "note": "e2e = lpsg_create (A upload from pinned host memory) + solve from the "
                   "start basis + x readback; solve = the reference's solve() clock boundary "
                   "(solver.cpp:332,363); max over ranks"}
    tto_reinv = None
    if world == 1 and cfg.get("reinv_every") and not args.no_reinversion:
        # the opt-in reinversion mode (include/lpsg.h reinvert_every): NOT the
        # reference's arithmetic, so it is reported beside the parity-mode
        # result, never as the headline; same API, host buffers, full solve
        cfg3 = solver_config(P, args, world, rank, local, reinvert_every=cfg["reinv_every"],
                             max_iter=args.e2e_max_iter)
        t0 = time.perf_counter()
        s3 = P.SimplexSolver(lp, cfg3)
        rep3 = s3.solve()
        t1 = time.perf_counter()
        st3 = s3.reinvert_stats()
        dev3 = s3.device_ms() / 1e3
        s3.close()
        import numpy as np
        x3 = rep3.x
        res3 = (float(np.abs(lp.A @ x3 - lp.b).max() / np.abs(lp.b).max())
                if rep3.status == P.SolveStatus.optimal else None)
        tto_reinv = {"status": rep3.status.name, "objective": rep3.objective,
                     "iterations_phase1": rep3.iterations_phase1,
                     "iterations_phase2": rep3.iterations_phase2,
                     "seconds_e2e": t1 - t0, "seconds_solve": rep3.total_seconds,
                     "seconds_device": dev3, "iterations_per_s_e2e": rep3.iterations / (t1 - t0),
                     "reinvert_every": cfg["reinv_every"], "rebuilds": st3["rebuilds"],
                     "newton_steps": st3["steps"], "rebuild_seconds": st3["seconds"],
                     "residual_before_last": st3["residual_before"],
                     "residual_after_last": st3["residual_after"],
                     "feasibility_residual": res3,
                     "note": "opt-in periodic reinversion on the device (B^-1 rebuilt from the basis "
                             "columns every reinvert_every pivots and before accepting an optimal / "
                             "unbounded outcome; csrc/reinvert.cu). Not bit-identical to the "
                             "reference, which never re-factorises; the parity-mode result is "
                             "time_to_optimal"}
    digest = lp_digest(lp.A, lp.b, lp.c, lp.col_kind)
    line = {
        "metric": METRIC, "value": value, "unit": "iterations/s", "n_gpus": world, "steps": done,
        "warmup": W, "ms_per_step": dev_ms / max(1, done), "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (reference generator lps::generate, seed 1)",
        "config": bench_config(cfg, lp.m, lp.n_total, digest, W, done),
        "parallelism": "single GPU" if world == 1 else
                       f"{world} shards: rows of B^-1 and pricing columns split, "
                       f"{'P2P (NVLink stores + flags)' if args.transport == 'p2p' else 'NCCL'} exchanges",
        "roofline": roofline,
        "e2e": e2e,
        "time_to_optimal": tto,
        "time_to_optimal_reinversion": tto_reinv,
        "gpu_launches": c1["kernel_launches"] - c0["kernel_launches"],
        "clocks": clk.summary(),
    }
    if exchange:
        line["exchange"] = exchange
    if (la_stats["bounded"] or la_stats["price_bounded"]) and world == 1:
        # transparency: the same window with the bounded lookahead off (every
        # tie scored by both exact GEMMs), the decisions being identical
        s2 = P.SimplexSolver(lp, solver_config(P, args, world, rank, local, max_iter=W,
                                               lookahead_bound="off"))
        s2.solve()
        s2.set_max_iter(W + K)
        rep2 = s2.solve()
        d2 = s2.device_ms()
        s2.close()
        la_stats["full_scoring_it_s"] = (rep2.iterations - W) / (d2 / 1e3) if d2 > 0 else None
    if any(la_stats.values()):
        line["lookahead"] = dict(la_stats, note=(
            "lookaheads of >= 16 candidates over the timed + profiled windows. bounded / full: "
            "select_leaving ties settled by the bounded selection (every later score provably "
            "<= the first survivor's +-0; the theta' GEMM skipped) vs scored in full. "
            "price_bounded / price_exact: pricings settled by the DMMA screen with rigorous "
            "error bounds + exact chains for the columns it cannot exclude vs the exact GEMM "
            "rerun. probe_rounds: selections whose DMMA probe screen left candidates for the "
            "exact probe rounds. full_scoring_it_s: the same window with lookahead_bound='off' "
            "(every tie scored by both exact GEMMs). Decisions are the reference's either way "
            "(DESIGN.md §4.1)"))
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cores = os.cpu_count() or 1
        kc = min(K, cfg["cpu_pivots"])
        Wc = W if W + kc <= cfg.get("ref_max_steps", 1 << 30) else 0
        val, n, secs, kind, used, w1 = reference_best(lp, Wc, kc, cfg)
        line["cpu_baseline"] = {"value": val, "unit": "iterations/s", "cores": used, "kind": kind,
                                "sample": f"pivots [{Wc}, {Wc + n}) of the same LP ({secs:.2f} s): "
                                          f"lps::two_phase_solve from oracle/_ref (unmodified "
                                          f"reference sources), best of workers = {cores} and "
                                          f"workers = 1 (here {used})"}
        if w1 is not None:
            line["cpu_baseline"]["workers_1"] = w1
        if val:
            # the reference's time to the same final status,
            # extrapolated as its measured time per pivot x the pivots of the
            # bit-identical GPU run (labelled as an extrapolation, not a run)
            piv = tto["iterations_phase1"] + tto["iterations_phase2"]
            line["cpu_baseline"]["extrapolated_time_to_status_s"] = {
                "status": tto["status"], "pivots": piv, "seconds": piv / val,
                "note": "extrapolated: measured CPU time per pivot x the GPU run's pivot count "
                        "(the pivot sequence is bit-identical)"}
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=1000)  # ~0.34 s timed at C3: several clock samples
    ap.add_argument("--warmup", type=int, default=20)
    ap.add_argument("--config", default="c3", choices=sorted(CONFIGS))
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--e2e-max-iter", type=int, default=0,
                    help="pivot budget of the end-to-end solve (0 = to optimality)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--batch", type=int, default=0, help="pivots per host check (0 = auto)")
    ap.add_argument("--transport", default="p2p", choices=["p2p", "nccl"],
                    help="N>1 exchanges: device-initiated NVLink stores + flags (p2p) or NCCL")
    ap.add_argument("--no-reinversion", action="store_true",
                    help="skip the opt-in reinversion-mode time-to-optimal solve")
    ap.add_argument("--no-profile", action="store_true",
                    help="no per-kernel CUDA events in the timed region (roofline omitted)")
    args = ap.parse_args()
    cfg = CONFIGS[args.config]
    if args.impl == "reference":
        run_reference_arm(args, cfg)
        return
    try:
        run_ours(args, cfg)
    except Exception as e:  # noqa: BLE001
        if int(os.environ.get("WORLD_SIZE", "1")) > 1 and args.transport == "p2p":
            # every rank fails the same exchange (it times out on all of them)
            print(f"bench: p2p transport failed ({e}); retrying with NCCL", file=sys.stderr, flush=True)
            args.transport = "nccl"
            run_ours(args, cfg)
        else:
            raise


if __name__ == "__main__":
    main()
