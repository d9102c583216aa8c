#!/usr/bin/env python
"""Benchmark of the Bit-GraphBLAS hot path on B200 (BASELINE.json configs[1]).

Step = one BFS (level-synchronous masked bin-SpMV sweeps, algorithms.py:75-93)
from one Graph500-style root on the undirected R-MAT scale-22 graph
(edge factor 16), graph and transpose resident in HBM.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

Prints ONE JSON line (rank 0):
  value      whole-job BFS GTEPS (undirected edges of the traversed component
             / device time; Graph500 convention, construction excluded)
  e2e        GTEPS through the public API with HOST inputs: H2D copy of the
             B2SR arrays, transpose, BFS, D2H of the levels, every step
  roofline   the K4 bin-SpMV kernel (masked full sweep, 50% random x) at the
             headline tile width: algorithmic bytes / CUDA-event kernel time
             vs MEASURED_PEAKS.json hbm_gbs
  cpu_baseline  the C oracle (oracle/, a restatement of the reference's CPU
             algorithm) on a bounded sample of the same workload
  sweep      per tile width: conversion, transpose, SpMV GB/s, BFS GTEPS
  tc         triangle counting (masked bin-SpGEMM) on R-MAT scale 20
Inputs (1 GB at d=4, 16 GB at d=32) exceed the 126 MB L2, so no flush is
needed between steps; the SpMV roofline loop flushes L2 explicitly anyway.
"""

from __future__ import annotations

import argparse
import ctypes
import json
import os
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "bin-SpMV GB/s vs HBM peak; BFS GTEPS and TC edges/s at 1/2/4/8 B200"


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=64)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--impl", choices=("ours", "reference"), default="ours")
    p.add_argument("--scale", type=int, default=22)
    p.add_argument("--edgefactor", type=int, default=16)
    p.add_argument("--dims", default="4,8,16,32", help="tile widths in the sweep")
    p.add_argument("--dim", type=int, default=4, help="headline tile width (0 = best of the sweep)")
    p.add_argument("--tc-scale", type=int, default=20)
    p.add_argument("--no-tc", action="store_true")
    p.add_argument("--no-cpu", action="store_true")
    p.add_argument("--drivers-scale", type=int, default=24, help="PR/SSSP/CC scale (BASELINE configs[3])")
    p.add_argument("--no-drivers", action="store_true")
    p.add_argument("--seed", type=int, default=1)
    p.add_argument("--workload", choices=("auto", "s22", "s26"), default="auto",
                   help="auto: configs[1] (s22 BFS) on one GPU, configs[4] (s26 strong scaling) under torchrun N>1")
    p.add_argument("--scale5", type=int, default=26, help="configs[4] graph scale")
    p.add_argument("--no-config5", action="store_true", help="skip the configs[4] N=1 point in the s22 run")
    return p.parse_args()


def peaks():
    try:
        return json.loads((ROOT / "MEASURED_PEAKS.json").read_text()), "measured"
    except Exception:
        return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0}, "fallback"


# ---------------------------------------------------------------- clocks
class Clocks:
    """NVML sampler (every 2 ms) of SM clock and clock-event reasons, running
    during the timed region; falls back to nvidia-smi -lms when NVML is absent."""

    REASONS = (("hw_slowdown", "nvmlClocksEventReasonHwSlowdown"),
               ("hw_thermal_slowdown", "nvmlClocksEventReasonHwThermalSlowdown"),
               ("sw_thermal_slowdown", "nvmlClocksEventReasonSwThermalSlowdown"),
               ("sw_power_cap", "nvmlClocksEventReasonSwPowerCap"),
               ("hw_power_brake", "nvmlClocksEventReasonHwPowerBrakeSlowdown"))

    def __init__(self, cuda_index: int):
        self.cuda_index, self.sm, self.reasons, self.max, self.errors = cuda_index, [], set(), None, set()
        self._stop = threading.Event()
        self.t = None

    def __enter__(self):
        try:
            import pynvml
            import torch

            pynvml.nvmlInit()
            idx = torch.cuda._get_nvml_device_index(self.cuda_index)
            self.nv, self.h = pynvml, pynvml.nvmlDeviceGetHandleByIndex(idx)
            self.max = float(pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM))
            self._sample()  # at the start of the region, whatever the thread's scheduling
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        except Exception:
            self.t = None
        return self

    def _sample(self):
        nv = self.nv
        self.sm.append(float(nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM)))
        try:
            r = nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
        except Exception:
            try:
                r = nv.nvmlDeviceGetCurrentClocksThrottleReasons(self.h)
            except Exception as e:
                self.errors.add(type(e).__name__)
                return
        for name, attr in self.REASONS:
            if r & getattr(nv, attr, 0):
                self.reasons.add(name)

    def _run(self):
        while not self._stop.is_set():
            try:
                self._sample()
            except Exception as e:
                self.errors.add(type(e).__name__)
            time.sleep(0.002)

    def __exit__(self, *a):
        if self.t:
            try:
                self._sample()  # and at its end
            except Exception as e:
                self.errors.add(type(e).__name__)
        self._stop.set()
        if self.t:
            self.t.join(timeout=2)
            if not self.sm:
                try:
                    self._sample()
                except Exception:
                    pass

    def summary(self):
        if not self.sm:
            return {"sm_mhz": None, "sm_max_mhz": self.max, "reasons": ["unsampled"]}
        out = {"sm_mhz": float(np.median(self.sm)), "sm_max_mhz": self.max, "reasons": sorted(self.reasons),
               "samples": len(self.sm), "source": "nvml, 2 ms"}
        if self.errors:
            out["nvml_errors"] = sorted(self.errors)
        return out


# ---------------------------------------------------------------- helpers
def pick_roots(deg: np.ndarray, k: int, seed: int):
    rng = np.random.default_rng(seed)
    cand = np.flatnonzero(deg > 0)
    return [int(v) for v in rng.choice(cand, size=min(k, len(cand)), replace=False)]


def traversed_edges(levels: np.ndarray, deg: np.ndarray) -> int:
    """Undirected edges inside the traversed component (Graph500 TEPS numerator)."""
    return int(deg[np.isfinite(levels)].sum() // 2)


def measured_traffic(kernel: str, scale: int, d: int):
    """dram__bytes_read.sum + dram__bytes_write.sum per launch of `kernel` from the
    committed ncu --set full capture (profiles/*_traffic.json), or None."""
    for f in sorted((ROOT / "profiles").glob("*_traffic.json"), reverse=True):
        try:
            for row in json.loads(f.read_text()):
                if row["kernel"] == kernel and row["scale"] == scale and row["tile_dim"] == d:
                    return row["dram_bytes"]
        except Exception:
            continue
    return None


def k4_time(_capi, dev, torch, h, xd, kd, yd, flush, sp, reps=10):
    """Masked K4 sweeps with an L2 flush before each: (mean streaming-kernel ms
    from the library's CUDA-event bracket on the launch stream, mean ms of the
    whole b2sr_bmv_bbb call incl. its small memset / hot-fill / keep kernels)."""
    _capi.call("b2sr_set_kernel_timing", 1)
    kt, ct = [], []
    ms = ctypes.c_float()
    for i in range(reps + 2):
        flush.zero_()
        a0, a1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a0.record()
        _capi.call("b2sr_bmv_bbb", h.ptr, dev.ptr(xd), dev.ptr(kd), dev.ptr(yd), sp)
        a1.record()
        torch.cuda.synchronize()
        _capi.call("b2sr_last_kernel_ms", ctypes.addressof(ms))
        if i >= 2:
            kt.append(ms.value)
            ct.append(a0.elapsed_time(a1))
    _capi.call("b2sr_set_kernel_timing", 0)
    return float(np.mean(kt)), float(np.mean(ct))


def bfs_byte_accounting(torch, at, lv, sweeps, d, bfs_ms, peak_gbs):
    """SURVEY.md §8d BFS byte accounting for one root (outside the timed
    region): per sweep L, the reference reads a full masked bbb sweep
    (kernels.py:219-225); a traversal NEEDS only the tile columns of tile rows
    whose keep word (~visited) is non-zero, the tile bytes of those tiles whose
    x word (the frontier) is non-zero, and the x / keep / y words.  Both
    totals over the BFS's sweeps (the final empty one included), and the
    needed bytes over the measured BFS time against the HBM peak."""
    wb = 4 if d == 32 else (2 if d == 16 else 1)
    tb = d * wb
    trp = torch.from_numpy(at.tile_row_ptr.astype(np.int64)).cuda()
    tci = torch.from_numpy(at.tile_col_ind.astype(np.int64)).cuda()
    ntr = trp.numel() - 1
    rows = torch.repeat_interleave(torch.arange(ntr, device="cuda"), trp[1:] - trp[:-1])
    lens = trp[1:] - trp[:-1]
    pad = torch.full((ntr * d,), float("inf"), dtype=torch.float64, device="cuda")
    pad[: lv.numel()] = lv
    lt = pad.view(ntr, d)
    vec = 3 * ntr * wb + 4 * (ntr + 1)
    needed = full = 0
    for L in range(1, sweeps + 1):
        keep = (lt >= L).any(dim=1)  # tile rows still holding an unvisited vertex (~visited != 0)
        front = (lt == L - 1).any(dim=1)  # tile columns whose frontier word is non-zero
        live_tiles = keep[rows]
        needed += vec + 4 * int(lens[keep].sum().item()) + tb * int((live_tiles & front[tci]).sum().item())
        full += vec + int(tci.numel()) * (4 + tb)
    del trp, tci, rows, pad
    needed_gbs = needed / bfs_ms / 1e6
    return {"needed_bytes": needed, "full_sweep_bytes": full, "sweeps": sweeps, "bfs_ms": round(bfs_ms, 4),
            "needed_gbs": round(needed_gbs, 1), "needed_frac_of_peak": round(needed_gbs / peak_gbs, 4),
            "full_sweep_equivalent_gbs": round(full / bfs_ms / 1e6, 1),
            "note": "one root; needed = tile columns of rows with a keep bit + tile bytes where the frontier "
                    "word is non-zero + vectors (SURVEY.md §8d); full = the reference's masked sweeps"}


def bmv_alg_bytes(ntr: int, T: int, d: int) -> int:
    """Full masked bbb sweep: tile_row_ptr + T*(4 + tile bytes) + x, keep, y words."""
    wb = 4 if d == 32 else (2 if d == 16 else 1)
    return 4 * (ntr + 1) + T * (4 + d * wb) + 3 * ntr * wb


# ---------------------------------------------------------------- our arm
def run_ours(args, rank, world, local_rank):
    import torch

    import paper_2201_08560_b200 as b2
    from paper_2201_08560_b200 import _capi, rmat
    from paper_2201_08560_b200 import _device as dev

    torch.cuda.set_device(local_rank)
    dist = None
    if world > 1:
        import torch.distributed as dist

        dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    stream = torch.cuda.current_stream()
    sp = stream.cuda_stream

    def ev():
        return torch.cuda.Event(enable_timing=True)

    def barrier():
        if dist is not None:
            dist.barrier()
        torch.cuda.synchronize()

    # ---- graph (device generator + device COO->CSR) ----
    t0 = time.time()
    csr = rmat.rmat_csr(args.scale, args.edgefactor, seed=args.seed)
    torch.cuda.synchronize()
    gen_s = time.time() - t0
    n = csr.n
    deg = np.diff(csr.row_ptr.astype(np.int64))
    roots = pick_roots(deg, args.warmup + args.steps + 8, seed=args.seed + 7)
    pk, pk_kind = peaks()

    # ---- tile-width sweep ----
    sweep = {}
    flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
    rng = np.random.default_rng(11)
    for d in [int(x) for x in args.dims.split(",") if x]:
        # conversion and transpose: the second of two calls (the first grows the
        # memory pool), CUDA events around the C-ABI call on its stream
        s0, s1 = ev(), ev()
        for _ in range(2):
            m = None
            torch.cuda.synchronize()
            s0.record()
            m = b2.csr_to_b2sr(csr, d)
            s1.record()
            torch.cuda.synchronize()
        conv_ms = s0.elapsed_time(s1)
        at = None
        for _ in range(2):
            at = None  # the previous result's memory goes back to the pool first
            torch.cuda.synchronize()
            s0.record()
            at = b2.formats.B2srMatrix._wrap(b2.formats._new_handle("b2sr_transpose", m.handle().ptr, sp))
            s1.record()
            torch.cuda.synchronize()
        tr_ms = s0.elapsed_time(s1)
        m._transpose = at
        h = at.handle()
        hA = m.handle()
        ntr, T = h.ntr, h.num_tiles
        # K4 masked full sweep, 50% random x and keep
        xw = b2.BitVector.from_bools(rng.random(n) < 0.5, d).words
        kw = b2.BitVector.from_bools(rng.random(n) < 0.5, d).words
        xd = dev.to_device(xw, dev.padded_vec_bytes(ntr, d))
        kd = dev.to_device(kw, dev.padded_vec_bytes(ntr, d))
        yd = dev.empty_bytes(dev.padded_vec_bytes(ntr, d))
        spmv_ms, spmv_call_ms = k4_time(_capi, dev, torch, h, xd, kd, yd, flush, sp, reps=6)
        ab = bmv_alg_bytes(ntr, T, d)
        # BFS from a few roots
        bt = []
        edges = 0
        lvd = dev.empty_bytes(8 * n)
        itc = ctypes.c_int64()
        _capi.call("b2sr_bfs", hA.ptr, h.ptr, roots[-1], dev.ptr(lvd), ctypes.addressof(itc), sp)  # warm plans
        for r in roots[:4]:
            b0, b1 = ev(), ev()
            b0.record()
            _capi.call("b2sr_bfs", hA.ptr, h.ptr, r, dev.ptr(lvd), ctypes.addressof(itc), sp)
            b1.record()
            torch.cuda.synchronize()
            bt.append(b0.elapsed_time(b1))
            edges += traversed_edges(dev.to_host(lvd, np.float64, n), deg)
        sb = int(b2.storage_bytes(m))
        conv_b = 4 * (n + 1) + 4 * int(csr.nnz) + sb  # CSR read + B2SR written
        sweep[d] = {"tiles": int(T), "b2sr_bytes": sb, "convert_ms": round(conv_ms, 3),
                    "convert_gbs": round(conv_b / conv_ms / 1e6, 1),
                    "convert_frac": round(conv_b / conv_ms / 1e6 / pk["hbm_gbs"], 3),
                    "transpose_ms": round(tr_ms, 3), "transpose_gbs": round(2 * sb / tr_ms / 1e6, 1),
                    "transpose_frac": round(2 * sb / tr_ms / 1e6 / pk["hbm_gbs"], 3),
                    "spmv_ms": round(spmv_ms, 4), "spmv_call_ms": round(spmv_call_ms, 4),
                    "spmv_gbs": round(ab / spmv_ms / 1e6, 1), "spmv_frac": round(ab / spmv_ms / 1e6 / pk["hbm_gbs"], 3),
                    "bfs_ms": round(float(np.mean(bt[1:] or bt)), 3),
                    "bfs_gteps": round(edges / (sum(bt) / 1e3) / 1e9, 3)}
        del m, at, h, hA
        torch.cuda.empty_cache()

    d = args.dim or max(sweep, key=lambda k: sweep[k]["bfs_gteps"])
    m = b2.csr_to_b2sr(csr, d)
    at = b2.b2sr_transpose(m)
    h = at.handle()
    hA = m.handle()
    b2sr_gb = b2.storage_bytes(m) / 1e9

    # ---- timed BFS steps (device-resident: graph, transpose, levels stay in HBM) ----
    n_steps = args.steps
    lev = [dev.empty_bytes(8 * n) for _ in range(n_steps)]
    it = ctypes.c_int64()
    for r in roots[: args.warmup]:
        _capi.call("b2sr_bfs", hA.ptr, h.ptr, r, dev.ptr(lev[0]), ctypes.addressof(it), sp)
    barrier()
    launches0 = _capi.launch_count()
    iters = []
    with Clocks(local_rank) as clk:
        marks = [ev() for _ in range(n_steps + 1)]  # per-root boundaries (same stream, no extra sync)
        marks[0].record()
        for k, r in enumerate(roots[args.warmup: args.warmup + n_steps]):
            _capi.call("b2sr_bfs", hA.ptr, h.ptr, r, dev.ptr(lev[k]), ctypes.addressof(it), sp)
            iters.append(int(it.value))
            marks[k + 1].record()
        barrier()
    e0, e1 = marks[0], marks[-1]
    launches = _capi.launch_count() - launches0
    ms = e0.elapsed_time(e1)
    degt = torch.from_numpy(deg).to("cuda")
    edges = 0
    per_root = []
    for k in range(n_steps):  # after the timed region: Graph500 edge count per root
        lv = lev[k].view(torch.float64)[:n]
        ek = int(degt[torch.isfinite(lv)].sum().item()) // 2
        edges += ek
        per_root.append(ek / (marks[k].elapsed_time(marks[k + 1]) / 1e3) / 1e9)
    gteps_hmean = len(per_root) / sum(1.0 / max(g, 1e-12) for g in per_root)
    bfs_bytes = bfs_byte_accounting(torch, at, lev[0].view(torch.float64)[:n], iters[0], d,
                                    marks[0].elapsed_time(marks[1]), peaks()[0]["hbm_gbs"])
    del lev
    if dist is not None:
        t = torch.tensor([ms], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
        e = torch.tensor([edges], device="cuda", dtype=torch.float64)
        dist.all_reduce(e)
        edges = int(e.item())
    value = edges / (ms / 1e3) / 1e9

    # ---- roofline of the K4 kernel at the headline width ----
    ntr, T = h.ntr, h.num_tiles
    xd = dev.to_device(b2.BitVector.from_bools(rng.random(n) < 0.5, d).words, dev.padded_vec_bytes(ntr, d))
    kd = dev.to_device(b2.BitVector.from_bools(rng.random(n) < 0.5, d).words, dev.padded_vec_bytes(ntr, d))
    yd = dev.empty_bytes(dev.padded_vec_bytes(ntr, d))
    kms, call_ms = k4_time(_capi, dev, torch, h, xd, kd, yd, flush, sp, reps=10)
    ab = bmv_alg_bytes(ntr, T, d)
    achieved = ab / kms / 1e6
    roofline = {"bound": "hbm", "kernel": f"k_bmv_bbb_stream<{d}> (masked full sweep, R-MAT s{args.scale})", "achieved": round(achieved, 1),
                "peak": pk["hbm_gbs"], "peak_kind": pk_kind, "unit": "GB/s", "frac": round(achieved / pk["hbm_gbs"], 4),
                "frac_of_8tbs_nominal": round(achieved / 8000.0, 4), "alg_bytes": ab,
                "traffic": measured_traffic(f"k_bmv_bbb_stream<{d}>", args.scale, d), "kernel_ms": round(kms, 4),
                "call_ms": round(call_ms, 4), "call_frac": round(ab / call_ms / 1e6 / pk["hbm_gbs"], 4),
                "timed": "CUDA events around the streaming kernel on its launch stream (b2sr_set_kernel_timing); "
                         "call_ms: the whole b2sr_bmv_bbb call incl. memset, hot fill and keep AND kernels"}

    # ---- e2e: public API with host inputs ----
    # the caller's B2srMatrix holds ordinary (pageable) numpy arrays; the
    # library stages the upload through its own page-locked chunks (staging.cu)
    host = (m.tile_row_ptr.copy(), m.tile_col_ind.copy(), m.bit_tiles.copy())
    hm = b2.B2srMatrix(n, d, *host)
    e2e_steps = max(3, min(args.steps, 6))
    e2e_edges = 0
    # untimed warm-up of the same loop (the result arrays are kept alive, as in
    # the timed loop, so the pinned result pool reaches its steady state)
    warm = [b2.bfs(_fresh(hm), r).per_vertex for r in roots[: max(args.warmup, e2e_steps)]]
    del warm
    barrier()
    f0, f1 = ev(), ev()
    outs = []
    f0.record()
    for r in roots[args.warmup: args.warmup + e2e_steps]:
        hm2 = _fresh(hm)  # no cached device mirror or transpose: H2D every step
        outs.append(b2.bfs(hm2, r).per_vertex)
    f1.record()
    barrier()
    e2e_ms = f0.elapsed_time(f1)
    e2e_edges = sum(traversed_edges(lv, deg) for lv in outs)
    del outs
    # phase breakdown of one extra call (not part of the value)
    ph = [ev() for _ in range(4)]
    hm2 = _fresh(hm)
    ph[0].record()
    hh = hm2.handle()
    ph[1].record()
    lvd = dev.empty_bytes(8 * n)
    _capi.call("b2sr_bfs", hh.ptr, None, roots[args.warmup], dev.ptr(lvd), ctypes.addressof(it), sp)
    ph[2].record()
    lv_host = dev.to_host(lvd, np.float64, n)
    ph[3].record()
    torch.cuda.synchronize()
    breakdown = {k: round(ph[i].elapsed_time(ph[i + 1]), 3) for i, k in enumerate(("h2d", "bfs", "d2h"))}
    del hh, hm2, lv_host
    e2e = {"value": round(e2e_edges / (e2e_ms / 1e3) / 1e9, 4), "unit": "GTEPS",
           "h2d_bytes_per_step": int(sum(a.nbytes for a in host)), "d2h_bytes_per_step": 8 * n,
           "ms_per_step": round(e2e_ms / e2e_steps, 3),
           "includes": "H2D of the B2SR arrays from the caller's pageable numpy arrays (staged by the library), "
                       "BFS (a fresh matrix has no transpose: push-only levels), D2H of the levels",
           "breakdown_ms": breakdown}

    # ---- TC on the scale-20 graph ----
    tc = None
    if not args.no_tc:
        tc = bench_tc(args, b2, rmat, torch, ev)
    drivers = None
    if not args.no_drivers:
        del m, at, h, hA
        torch.cuda.empty_cache()
        drivers = bench_drivers(args, b2, rmat, torch, ev)

    line = {"metric": METRIC, "value": round(value, 4), "unit": "GTEPS", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": round(ms / args.steps, 4), "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "u32 bit-words (b1 tiles)",
            "data": f"synthetic R-MAT (Graph500 a,b,c=.57,.19,.19) generated on device, seed {args.seed}",
            "config": workload_config("s22", args, args.scale, n, int(csr.nnz), d, world, int(b2sr_gb * 1e9)),
            "e2e": e2e, "roofline": roofline, "gpu_launches": int(launches), "bfs_sweeps_per_root": iters[:4],
            "gteps_harmonic_mean": round(gteps_hmean, 4), "bfs_bytes": bfs_bytes,
            "clocks": clk.summary(), "sweep": {str(k): v for k, v in sweep.items()}, "tc": tc, "drivers": drivers,
            "graph_gen_s": round(gen_s, 3)}
    if rank == 0 and world == 1 and not args.no_cpu:
        line["cpu_baseline"], lv_cpu = cpu_baseline(csr, d, roots[args.warmup])
        # parity of the headline: the oracle's levels for that root vs the device's
        lv_gpu = b2.bfs(b2.csr_to_b2sr(csr, d), roots[args.warmup]).per_vertex
        line["parity"] = {"bfs_levels_vs_oracle": bool(lv_gpu.tobytes() == lv_cpu.tobytes()),
                          "root": roots[args.warmup],
                          "full_size_tests": "tests/test_gpu_configs.py (configs 0-3 vs the oracle)"}
    if not args.no_config5:
        del csr
        torch.cuda.empty_cache()
        line["config5_n1"] = run_strong(args, 0, 1, local_rank, tdist=None, headline=False)
    if rank == 0:
        print(json.dumps(line), flush=True)
    if dist is not None:
        dist.destroy_process_group()


def _fresh(hm):
    """Same host arrays, no device mirror (forces the H2D copy)."""
    import copy

    import threading

    c = copy.copy(hm)
    c._lock = threading.RLock()
    c._h = None
    c._transpose = None
    c._nodiag = None
    c._bfs_push = 0
    return c


def bench_drivers(args, b2, rmat, torch, ev):
    """BASELINE configs[3]: PageRank (10 iterations), SSSP and CC on R-MAT
    scale 24 through the public API (parity vs the C oracle: tools/config4.py)."""
    csr = rmat.rmat_csr(args.drivers_scale, args.edgefactor, seed=args.seed)
    d = 4
    m = b2.csr_to_b2sr(csr, d)
    at = b2.b2sr_transpose(m)
    deg = np.diff(csr.row_ptr.astype(np.int64)).astype(np.float64)
    src = int(np.argmax(deg))
    out = {"scale": args.drivers_scale, "tile_dim": d, "nnz": int(csr.nnz), "tiles": int(m.num_tiles)}

    def timed(fn):
        fn()  # warm (work partitions, long-row lists)
        a0, a1 = ev(), ev()
        a0.record()
        r = fn()
        a1.record()
        torch.cuda.synchronize()
        return r, a0.elapsed_time(a1)

    r, ms = timed(lambda: b2.pagerank(at, deg))
    out["pagerank"] = {"ms": round(ms, 3), "iterations": r.iterations, "ms_per_iter": round(ms / r.iterations, 3),
                       "mode": "exact (bit-identical to the reference)"}
    os.environ["B2SR_PR_MODE"] = "fast"  # documented tolerance mode (relative L1 <= 1e-5)
    try:
        rf, msf = timed(lambda: b2.pagerank(at, deg))
    finally:
        del os.environ["B2SR_PR_MODE"]
    out["pagerank_fast"] = {"ms": round(msf, 3), "iterations": rf.iterations, "ms_per_iter": round(msf / rf.iterations, 3),
                            "rel_l1_vs_exact": float(np.abs(rf.per_vertex - r.per_vertex).sum() / np.abs(r.per_vertex).sum()),
                            "mode": "B2SR_PR_MODE=fast: float32 x (L2-resident), float64 order-free sums"}
    r, ms = timed(lambda: b2.sssp(m, src))
    out["sssp"] = {"ms": round(ms, 3), "iterations": r.iterations}
    r, ms = timed(lambda: b2.connected_components(m))
    out["cc"] = {"ms": round(ms, 3), "iterations": r.iterations}
    return out


def bench_tc(args, b2, rmat, torch, ev):
    """BASELINE configs[2]: triangle counting on R-MAT scale 20 through the
    masked bin-SpGEMM.  Besides the end-to-end count time, the SpGEMM kernel
    is timed alone (CUDA events on its stream) and its AND+POPC work W is
    counted, for W/t against the measured AND+POPC peak."""
    from paper_2201_08560_b200 import _capi

    csr = rmat.rmat_csr(args.tc_scale, args.edgefactor, seed=args.seed)
    out = {}
    try:
        popc_peak = json.loads((ROOT / "profiles" / "r01_popc_peak.json").read_text())["and_popc_units_per_s"]
    except Exception:
        popc_peak = 148 * 16 * 1.965e9
    dag = b2.algorithms._degree_oriented(csr)  # what triangle_count() feeds the masked SpGEMM
    for d in (4, 8):
        lo = b2.csr_to_b2sr(dag, d)
        h = lo.handle()
        cnt, work, kms_ = ctypes.c_int64(), ctypes.c_uint64(), ctypes.c_float()
        _capi.call("b2sr_tc_work", h.ptr, ctypes.addressof(cnt), ctypes.addressof(work), 0)
        b2.algorithms._tc_count(lo)  # warm
        ts, ks = [], []
        _capi.call("b2sr_set_kernel_timing", 1)
        for _ in range(3):
            e0, e1 = ev(), ev()
            e0.record()
            c = b2.algorithms._tc_count(lo)
            e1.record()
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1))
            _capi.call("b2sr_last_kernel_ms", ctypes.addressof(kms_))
            ks.append(kms_.value)
        _capi.call("b2sr_set_kernel_timing", 0)
        ms, kms = float(np.median(ts)), float(np.median(ks))
        assert c == cnt.value
        out[str(d)] = {"triangles": int(c), "ms": round(ms, 3), "edges_per_s": round((csr.nnz // 2) / (ms / 1e3), 1),
                       "lower_tiles": int(lo.num_tiles), "spgemm_kernel_ms": round(kms, 3),
                       "work_units": int(work.value), "units_per_s": round(work.value / (kms / 1e3), 1),
                       "popc_peak_units_per_s": popc_peak,
                       "popc_frac": round(work.value / (kms / 1e3) / popc_peak, 4)}
    return {"scale": args.tc_scale, "nnz": int(csr.nnz), "by_tile_dim": out,
            "kernel": "k_tc_filter (each pair of L staged on its longer row: shared-memory filter probes, "
                      "queued hits, AND+POPC) + k_bmm_masked_items for rows over 1024 tiles: sum over the "
                      "degree-oriented DAG L of (L L^T) (= triangles; the reference uses the ID-ordered lower triangle)",
            "note": "work_units = AND+POPC units W; ms = the whole b2sr_tc call (incl. the transpose of L), "
                    "spgemm_kernel_ms = the masked SpGEMM kernels; bound by probe issue, not POPC"}


def cpu_baseline(csr, d, root):
    """C oracle BFS (transpose + masked sweeps, OpenMP over tile rows) on the same graph."""
    from oracle import oracle as orc

    n = csr.n
    rp, ci = csr.row_ptr, csr.col_ind
    threads = os.cpu_count() or 1
    m = orc.csr_to_b2sr(n, rp, ci, d)
    t0 = time.perf_counter()
    lv, it = orc.bfs(m, root, workers=threads)
    dt = time.perf_counter() - t0
    deg = np.diff(rp.astype(np.int64))
    e = traversed_edges(lv, deg)
    return {"value": round(e / dt / 1e9, 6), "unit": "GTEPS", "cores": threads, "kind": "port",
            "sample": f"1 BFS root (transpose included, as bfs() does) on the same scale graph, B2SR-{d}",
            "seconds": round(dt, 3)}, lv


def cpu_baseline_s26(args):
    """configs[4] at N=1: the C oracle on the same s26 graph (its CSR copied
    down from the device), one root, the undirected matrix as its own
    transpose (SURVEY.md §8c restatement rule; the transpose alone would
    dominate)."""
    from oracle import oracle as orc

    from paper_2201_08560_b200 import rmat

    d = args.dim or 4
    csr = rmat.rmat_csr(args.scale5, args.edgefactor, seed=args.seed)
    n, rp, ci = csr.n, csr.row_ptr, csr.col_ind
    del csr
    threads = os.cpu_count() or 1
    t0 = time.perf_counter()
    m = orc.csr_to_b2sr(n, rp, ci, d, workers=threads)
    conv = time.perf_counter() - t0
    deg = np.diff(rp.astype(np.int64))
    root = pick_roots(deg, args.warmup + args.steps + 8, seed=args.seed + 7)[args.warmup]
    t0 = time.perf_counter()
    lv, _ = orc.bfs(m, root, workers=threads, symmetric=True)
    dt = time.perf_counter() - t0
    return {"value": round(traversed_edges(lv, deg) / dt / 1e9, 6), "unit": "GTEPS", "cores": threads, "kind": "port",
            "sample": f"1 BFS root on the same s{args.scale5} graph, B2SR-{d}, matrix as its own transpose",
            "seconds": round(dt, 3), "oracle_convert_s": round(conv, 2)}


# ---------------------------------------------------------------- configs[4]: strong scaling
def run_strong(args, rank, world, local_rank, tdist=None, headline=True):
    """BASELINE configs[4]: row-partitioned BFS + TC on undirected R-MAT scale
    26 (B2SR-4) over N GPUs -- strong scaling, the same graph and the same
    native driver (b2sr_dist_bfs_*, NCCL) at every N including 1.  Each rank
    builds the graph on its GPU, cuts its rows of a and at (balanced by at's
    tiles) and drops the rest; per level the ranks exchange row contributions
    (all-to-all-v) and the merged rows (all-gather-v) inside the library.
    value = traversed edges of the whole job / max-over-ranks device time.
    Returns the JSON line (headline) or a summary dict."""
    import torch

    import paper_2201_08560_b200 as b2
    from paper_2201_08560_b200 import _capi, rmat
    from paper_2201_08560_b200 import _device as dev
    from paper_2201_08560_b200 import dist as bdist

    sp = torch.cuda.current_stream().cuda_stream
    ev = lambda: torch.cuda.Event(enable_timing=True)  # noqa: E731

    def barrier():
        if tdist is not None:
            tdist.barrier()
        torch.cuda.synchronize()

    def max_over_ranks(v):
        if tdist is None:
            return float(v)
        t = torch.tensor([float(v)], device="cuda", dtype=torch.float64)
        tdist.all_reduce(t, op=tdist.ReduceOp.MAX)
        return float(t.item())

    scale, d = args.scale5, args.dim or 4
    t0 = time.time()
    csr = rmat.rmat_csr(scale, args.edgefactor, seed=args.seed)
    n, nnz = csr.n, int(csr.nnz)
    deg = np.diff(csr.row_ptr.astype(np.int64))
    m = b2.csr_to_b2sr(csr, d)
    at = b2.b2sr_transpose(m)
    b2sr_bytes = int(b2.storage_bytes(m))
    comm = bdist.Comm.from_torch(tdist) if tdist is not None else bdist.Comm.nccl_single()
    plan = bdist.NativeDistributedBfs.from_matrices(comm, m, at)
    rb, re_ = plan.rows
    # this rank's rows as the caller's host arrays (pageable numpy), for the e2e leg
    blk_a = b2.formats._new_handle("b2sr_row_block", m.handle().ptr, rb, re_, sp)
    blk_at = b2.formats._new_handle("b2sr_row_block", at.handle().ptr, rb, re_, sp)
    host_a, host_at = bdist.block_to_host(blk_a, pinned=False), bdist.block_to_host(blk_at, pinned=False)
    trp_a, trp_at = m.tile_row_ptr.copy(), at.tile_row_ptr.copy()
    del blk_a, m, at
    torch.cuda.empty_cache()
    setup_s = time.time() - t0
    roots = pick_roots(deg, args.warmup + args.steps + 8, seed=args.seed + 7)
    degt = torch.from_numpy(deg).to("cuda")
    lev = dev.empty_bytes(8 * n)
    for r in roots[: args.warmup]:
        plan.run(r, to_host=False, levels=lev)
    barrier()
    launches0 = _capi.launch_count()
    iters, edges = [], 0
    t_total = 0.0
    with Clocks(local_rank) as clk:
        for r in roots[args.warmup: args.warmup + args.steps]:
            e0, e1 = ev(), ev()
            e0.record()
            _, it = plan.run(r, to_host=False, levels=lev)
            e1.record()
            torch.cuda.synchronize()
            t_total += e0.elapsed_time(e1)
            iters.append(it)
            lv = lev.view(torch.float64)[:n]
            edges += int(degt[torch.isfinite(lv)].sum().item()) // 2  # outside the timed region
        barrier()
    launches = _capi.launch_count() - launches0
    ms = max_over_ranks(t_total)
    value = edges / (ms / 1e3) / 1e9

    # K4 roofline of rank 0's block of at (masked sweep, 50 % random x / keep)
    roofline = None
    if rank == 0:
        pk, pk_kind = peaks()
        rng = np.random.default_rng(11)
        gb = dev.padded_vec_bytes(-(-n // d), d)
        xd = dev.to_device(b2.BitVector.from_bools(rng.random(n) < 0.5, d).words, gb)
        kd = dev.to_device(b2.BitVector.from_bools(rng.random(n) < 0.5, d).words, gb)
        yd = dev.empty_bytes(dev.padded_vec_bytes(blk_at.ntr, d) + 16)
        flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
        kms, call_ms = k4_time(_capi, dev, torch, blk_at, xd, kd, yd, flush, sp, reps=8)
        ab = bmv_alg_bytes(blk_at.ntr, blk_at.num_tiles, d)
        roofline = {"bound": "hbm", "kernel": f"k_bmv_bbb_stream<{d}> (masked sweep of rank 0's rows of at, s{scale})",
                    "achieved": round(ab / kms / 1e6, 1), "peak": pk["hbm_gbs"], "peak_kind": pk_kind, "unit": "GB/s",
                    "frac": round(ab / kms / 1e6 / pk["hbm_gbs"], 4), "alg_bytes": ab,
                    "traffic": measured_traffic(f"k_bmv_bbb_stream<{d}>", scale, d), "kernel_ms": round(kms, 4),
                    "call_ms": round(call_ms, 4),
                    "timed": "CUDA events around the streaming kernel on its launch stream (b2sr_set_kernel_timing)"}
        del xd, kd, yd, flush
    del blk_at
    torch.cuda.empty_cache()

    # e2e: every rank uploads its rows of a and at from pageable host arrays
    # (+ the global tile_row_ptr), plans, runs; rank 0 reads the levels back
    e2e_steps = 2
    barrier()
    f0, f1 = ev(), ev()
    f0.record()
    e2e_edges = 0
    for r in roots[args.warmup: args.warmup + e2e_steps]:
        ha = bdist.block_from_host(n, d, rb, re_, host_a)
        hat = bdist.block_from_host(n, d, rb, re_, host_at)
        p2 = bdist.NativeDistributedBfs.from_blocks(comm, ha, hat, trp_a, trp_at)
        lv, _ = p2.run(r, to_host=(rank == 0))
        if rank == 0:
            e2e_edges += traversed_edges(lv, deg)
        del p2, ha, hat, lv
    f1.record()
    barrier()
    e2e_ms = max_over_ranks(f0.elapsed_time(f1))
    h2d = sum(int(h[1].nbytes) for h in host_a + host_at) + trp_a.nbytes + trp_at.nbytes
    if tdist is not None:
        t = torch.tensor([h2d], device="cuda", dtype=torch.float64)
        tdist.all_reduce(t)
        h2d = int(t.item())
    del plan, lev, host_a, host_at
    torch.cuda.empty_cache()

    # TC: L (degree-oriented DAG) replicated, mask rows cut by estimated work
    tc = None
    if not args.no_tc:
        lower = b2.csr_to_b2sr(b2.algorithms._degree_oriented(csr), d)
        bdist.native_triangle_count(comm, lower)  # warm (plans)
        barrier()
        t0_, t1_ = ev(), ev()
        t0_.record()
        tri, cuts = bdist.native_triangle_count(comm, lower)
        t1_.record()
        barrier()
        tms = max_over_ranks(t0_.elapsed_time(t1_))
        tc = {"scale": scale, "nnz": nnz, "triangles": int(tri), "ms": round(tms, 3),
              "edges_per_s": round((nnz // 2) / (tms / 1e3), 1), "edges_per_s_per_gpu": round((nnz // 2) / (tms / 1e3) / world, 1),
              "mask_row_cuts": cuts, "lower_tiles": int(lower.num_tiles),
              "parallelism": f"mask tile rows x{world} (equal estimated work), L and L^T replicated, each pair counted by the owner of its longer row, NCCL int64 all-reduce"}
        del lower
    del csr
    torch.cuda.empty_cache()
    e2e = {"value": round(e2e_edges / (e2e_ms / 1e3) / 1e9, 4), "unit": "GTEPS", "h2d_bytes_per_step": h2d,
           "d2h_bytes_per_step": 8 * n, "ms_per_step": round(e2e_ms / e2e_steps, 3),
           "includes": "every rank: H2D of its rows of a and at from pageable numpy arrays (staged by the "
                       "library) + the global tile_row_ptr, plan, distributed BFS; D2H of the levels on rank 0"}
    summary = {"workload": f"row-partitioned BFS, undirected R-MAT scale {scale} edgefactor {args.edgefactor}, "
                           f"B2SR-{d}, strong scaling", "scale": scale, "n": n, "nnz": nnz, "tile_dim": d,
               "n_gpus": world, "bfs_gteps": round(value, 4), "per_gpu_gteps": round(value / world, 4),
               "ms_per_root": round(ms / args.steps, 4), "roots": args.steps, "bfs_sweeps_per_root": iters[:4],
               "rows": [rb, re_], "tc": tc, "roofline": roofline, "e2e": e2e, "setup_s": round(setup_s, 2),
               "b2sr_bytes": b2sr_bytes}
    if not headline:
        return summary
    line = {"metric": METRIC, "value": round(value, 4), "unit": "GTEPS", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": round(ms / args.steps, 4), "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "u32 bit-words (b1 tiles)",
            "data": f"synthetic R-MAT (Graph500 a,b,c=.57,.19,.19) generated on device, seed {args.seed}",
            "config": workload_config("s26", args, scale, n, nnz, d, world, b2sr_bytes),
            "e2e": e2e, "roofline": roofline, "gpu_launches": int(launches), "bfs_sweeps_per_root": iters[:4],
            "per_gpu_gteps": round(value / world, 4), "clocks": clk.summary(), "tc": tc,
            "setup_s": round(setup_s, 2)}
    return line


def run_dist(args, rank, world, local_rank):
    """torchrun entry (N >= 1 processes, one GPU each) of the configs[4] workload."""
    import torch
    import torch.distributed as tdist

    torch.cuda.set_device(local_rank)
    tdist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    line = run_strong(args, rank, world, local_rank, tdist=tdist, headline=True)
    if rank == 0:
        if world == 1 and not args.no_cpu:
            line["cpu_baseline"] = None  # the s26 CPU leg is the --impl reference arm
        print(json.dumps(line), flush=True)
    tdist.destroy_process_group()


# ---------------------------------------------------------------- reference arm
def run_reference(args, rank, world, workload):
    """The reference algorithm on host cores: the C restatement in oracle/ (the
    reference is pure Python/numpy and cannot travel), on our
    arm's workload (s22 at one GPU, s26 for the strong-scaling runs), its
    BFS transposing per call as algorithms.py:78 does."""
    if rank != 0:
        return
    from oracle import oracle as orc

    threads = os.cpu_count() or 1
    t0 = time.perf_counter()
    scale = args.scale5 if workload == "s26" else args.scale
    rp, ci = orc.rmat_csr(scale, args.edgefactor, seed=args.seed)
    n = 1 << scale
    d = args.dim or 4
    m = orc.csr_to_b2sr(n, rp, ci, d, workers=threads)
    setup = time.perf_counter() - t0
    deg = np.diff(rp.astype(np.int64))
    roots = pick_roots(deg, args.warmup + args.steps + 8, seed=args.seed + 7)
    budget_s = 150.0
    warm = args.warmup if workload == "s22" else 0  # s26: one root already takes about a minute
    for r in roots[:warm]:  # untimed warm-up roots (page-in, thread pool)
        orc.bfs(m, r, workers=threads)
    edges, secs, done = 0, 0.0, 0
    for r in roots[args.warmup: args.warmup + args.steps]:
        t1 = time.perf_counter()
        lv, _ = orc.bfs(m, r, workers=threads)
        secs += time.perf_counter() - t1
        edges += traversed_edges(lv, deg)
        done += 1
        if secs > budget_s:
            break
    v = edges / secs / 1e9
    tb = d * (4 if d == 32 else 2 if d == 16 else 1)
    b2sr_bytes = 4 * (len(m[2])) + len(m[3]) * (4 + tb)
    cfg = workload_config(workload, args, scale, n, int(len(ci)), d, world, b2sr_bytes)
    line = {"impl": "reference", "metric": METRIC, "value": round(v, 6), "unit": "GTEPS", "n_gpus": world,
            "steps": done, "warmup": warm, "ms_per_step": round(1e3 * secs / done, 2),
            "higher_is_better": True, "scaling": "strong" if workload == "s26" else "weak", "vs_baseline": None,
            "dtype": "u32 bit-words (b1 tiles)",
            "data": f"synthetic R-MAT (Graph500 a,b,c=.57,.19,.19), seed {args.seed} (CPU twin of the device generator)",
            "config": cfg,
            "cpu_baseline": {"value": round(v, 6), "unit": "GTEPS", "cores": threads, "kind": "port",
                             "sample": f"{done} BFS roots incl. the per-call transpose (timed budget {budget_s:.0f} s)"},
            "e2e": {"value": round(v, 6), "unit": "GTEPS", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
            "setup_s": round(setup, 2)}
    print(json.dumps(line), flush=True)


def workload_config(workload, args, scale, n, nnz, d, world, b2sr_bytes):
    """The config dict both arms print for a workload (identical keys and values)."""
    if workload == "s26":
        return {"workload": f"row-partitioned BFS, undirected R-MAT scale {scale} edgefactor {args.edgefactor}, "
                            f"B2SR-{d}, strong scaling", "scale": scale, "n": n, "nnz": nnz, "tile_dim": d,
                "roots": args.steps,
                "parallelism": f"row-partitioned x{world}: a/at tile-row blocks balanced by tiles, "
                               "all-to-all-v + all-gather-v of frontier words per level (NCCL)",
                "l2": "inputs larger than L2 (B2SR %.2f GB)" % (b2sr_bytes / 1e9)}
    return {"workload": f"BFS via masked bin-SpMV, undirected R-MAT scale {scale} edgefactor {args.edgefactor}, "
                        f"B2SR-{d}", "scale": scale, "n": n, "nnz": nnz, "tile_dim": d, "roots": args.steps,
            "parallelism": "single",
            "l2": "inputs larger than L2 (B2SR %.2f GB > 126 MB)" % (b2sr_bytes / 1e9)}


def main():
    args = parse()
    rank = int(os.environ.get("RANK", 0))
    world = int(os.environ.get("WORLD_SIZE", 1))
    local_rank = int(os.environ.get("LOCAL_RANK", 0))
    workload = args.workload if args.workload != "auto" else ("s26" if world > 1 else "s22")
    if args.impl == "reference":
        run_reference(args, rank, world, workload)
        return
    if workload == "s26":
        if "MASTER_ADDR" in os.environ:
            run_dist(args, rank, world, local_rank)
        else:  # one GPU without torchrun: the same native driver, NCCL world of one
            import torch

            torch.cuda.set_device(local_rank)
            line = run_strong(args, 0, 1, local_rank, tdist=None, headline=True)
            if not args.no_cpu:
                line["cpu_baseline"] = cpu_baseline_s26(args)
            print(json.dumps(line), flush=True)
        return
    run_ours(args, rank, world, local_rank)


if __name__ == "__main__":
    main()
