#!/usr/bin/env python
"""Benchmark of the B200 RPD hot path (BASELINE.json metric: tet-sphere pairs clipped/s and
full/partial RPD ms at 1/2/4/8 B200).

One step = one pass of the hot path over the bench workload:
full RPD of the C3 sphere set (stage + Alg. 1 filter + k_tet compaction + clip + piece
output), then the C4 partial updates (10 iterations inserting M = 500 spheres each,
re-filtering and re-clipping only touched tets), and with N > 1 GPUs the NCCL all-gather of
the pieces.  Tets are sharded block-cyclically over the ranks; spheres are replicated.

value = candidate (tet, sphere) pairs clipped per second by the whole job (all ranks, full +
partial), device time (CUDA events, max over ranks), inputs resident in HBM.
Usage: python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
"""
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

MEASURED = os.path.join(ROOT, "MEASURED_PEAKS.json")
FP64_PEAK = os.path.join(ROOT, "profiles", "fp64_peak.json")
NCU_TRAFFIC = os.path.join(ROOT, "profiles", "ncu_traffic.json")

WORKLOADS = {
    "C4": ("C3+C4: ~200k-tet box-with-hole Kuhn mesh, 20k medial-like spheres full RPD "
           "+ 10 partial updates x M=500 (final 25.5k spheres)"),
    "C3": "C3: ~200k-tet box-with-hole Kuhn mesh, 20k medial-like spheres, full RPD",
    "C5": ("C5: ~4M-tet box-with-hole Kuhn mesh, 50k medial-like spheres with high radius "
           "variance, full RPD"),
    "C2": "C2: ~50k-tet box-with-hole Kuhn mesh, 2k medial-like spheres, full RPD",
}


def workload_name(cfg):
    return WORKLOADS.get(cfg, cfg)


def bench_config(args, w, world):
    """The line's `config` (both arms: the reference arm runs the same workload)."""
    batches = w.batches if args.partial_iters < 0 else w.batches[:args.partial_iters]
    return {"workload": workload_name(args.config), "config": args.config, "T": w.T, "N": w.N,
            "partial_iters": len(batches), "M": (len(batches[0][0]) - w.N) if batches else 0,
            "filter": args.filter, "parallelism": f"tet-shard x{world}", "seed": args.seed,
            "l2": "flushed (256 MB write) before every timed step"}


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="C4", choices=sorted(WORKLOADS),
                    help="C4 (default): C3 full RPD + 10 partial updates; C5: 4M tets, 50k spheres")
    ap.add_argument("--filter", default="pruned", choices=["all_pairs", "pruned"])
    ap.add_argument("--partial-iters", type=int, default=-1,
                    help="partial updates per step (-1: all batches of the config)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-nbr", action="store_true",
                    help="skip the NEXT-3 side record (sphere neighbour lists on the GPU)")
    ap.add_argument("--no-small", action="store_true",
                    help="skip the M = 1 / M = 10 partial-update latency side measurement")
    ap.add_argument("--no-euler", action="store_true",
                    help="skip the fractional-Euler (NEXT-1) side measurement")
    ap.add_argument("--cpu-seconds", type=float, default=12.0)
    ap.add_argument("--seed", type=int, default=0,
                    help="workload seed (SURVEY.md §8(d): seeds 0, 1, 2 per config, median "
                         "reported; tools/seeds.py runs all three)")
    ap.add_argument("--force-shard", action="store_true",
                    help="run the sharded path (exchanges over a process group) even with one "
                         "rank, e.g. under torch.distributed.run --nproc-per-node 1 (testing)")
    return ap.parse_args()


# ----------------------------------------------------------------------------- helpers


class ClockSampler:
    """nvidia-smi clocks and throttle reasons sampled during the timed region."""
    FIELDS = ["clocks.sm", "clocks.max.sm", "clocks_event_reasons.hw_slowdown",
              "clocks_event_reasons.hw_thermal_slowdown",
              "clocks_event_reasons.sw_thermal_slowdown", "clocks_event_reasons.sw_power_cap"]
    NAMES = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]

    def __init__(self, device):
        self.device = device
        self.rows = []
        self.proc = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.device), "--query-gpu=" + ",".join(self.FIELDS),
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([x.strip() for x in line.split(",")])

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.25)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        sm = [float(r[0]) for r in self.rows if len(r) >= 6 and r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if len(r) >= 6 and r[1].replace(".", "").isdigit()]
        reasons = set()
        for r in self.rows:
            if len(r) >= 6:
                for k, name in enumerate(self.NAMES):
                    if r[2 + k] == "Active":
                        reasons.add(name)
        return {"sm_mhz": float(np.median(sm)) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": sorted(reasons),
                "samples": len(sm)}


def fp64_peak_tflops():
    """Measured DFMA peak (tools/fp64_peak.cu, committed under profiles/), else the nominal
    148 SMs x 64 DFMA/clk x 2 flop x 1.965 GHz."""
    try:
        d = json.load(open(FP64_PEAK))
        return float(d["fp64_tflops"]), "measured (profiles/fp64_peak.json, tools/fp64_peak.cu)"
    except Exception:
        return 148 * 64 * 2 * 1.965e9 / 1e12, "nominal 148x64x2x1.965GHz (no measurement found)"


def hbm_peak_gbs():
    try:
        return float(json.load(open(MEASURED))["hbm_gbs"]), "measured (MEASURED_PEAKS.json)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md)"


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


# ----------------------------------------------------------------------------- reference arm


def run_reference(args):
    """The oracle (plain CPU implementation, as it stands) on the host cores, on a bounded
    sample of the same workload per step (reference arm)."""
    world, rank, _ = dist_env()
    if world > 1 and rank != 0:
        return
    import oracle
    import rpd_workloads as W
    w = W.make_config(args.config, seed=args.seed)
    cores = oracle.max_threads()
    rng = np.random.default_rng(0)
    # calibrate the sample so the whole run ends in a few minutes
    per_tet = _oracle_per_tet(oracle, w, rng)
    budget = 150.0 / max(args.steps + args.warmup, 1)
    n_s = int(min(max(budget / max(per_tet, 1e-6), 16), w.T))
    times, pairs = [], []
    for s in range(args.warmup + args.steps):
        ids = np.sort(np.random.default_rng(100 + s).choice(w.T, n_s, replace=False)).astype(np.int32)
        t0 = time.perf_counter()
        r = oracle.rpd_workload(w, tet_ids=ids)
        dt = time.perf_counter() - t0
        if s >= args.warmup:
            times.append(dt)
            pairs.append(len(r["cand_idx"]))
    value = float(np.sum(pairs) / np.sum(times))
    sample = (f"{n_s} random tets per step of the {args.config} mesh (T={w.T}), full Alg. 1 over "
              f"all N={w.N} spheres + clip of their candidates")
    line = {"metric": "tet-sphere pairs clipped/s", "value": value, "unit": "pairs/s",
            "impl": "reference", "n_gpus": args.gpus, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": 1e3 * float(np.mean(times)),
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic", "config": bench_config(args, w, max(world, 1)),
            "cpu_baseline": {"value": value, "unit": "pairs/s", "cores": cores,
                             "kind": "oracle", "sample": sample},
            "e2e": {"value": value, "unit": "pairs/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def _oracle_per_tet(oracle, w, rng):
    """Oracle seconds per tet: two probe sizes, so that the per-call input validation (a pass
    over the whole mesh) cancels; if timing noise makes the difference vanish, the larger
    probe's average (an over-estimate, so the sample only gets smaller)."""
    ts, ns = [], (256, 2048)
    for n in ns:
        ids = np.sort(rng.choice(w.T, min(n, w.T), replace=False)).astype(np.int32)
        t0 = time.perf_counter()
        oracle.rpd_workload(w, tet_ids=ids)
        ts.append(time.perf_counter() - t0)
    d = (ts[1] - ts[0]) / (ns[1] - ns[0])
    return d if d > 0.2 * ts[1] / ns[1] else ts[1] / ns[1]


def cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    import platform
    return platform.processor() or platform.machine()


def cpu_baseline(w, seconds):
    """The oracle timed on a bounded sample of the bench workload (rank 0, N = 1), as it
    stands: all host cores and 1 thread, the Alg. 1 filter alone (clip=False) and the full
    RPD (filter + clip), so the clip's share is their difference (SURVEY.md §8(d) "Oracle
    timing"; BASELINE.md CPU-baseline plan)."""
    import oracle
    cores = oracle.max_threads()
    rng = np.random.default_rng(1)
    per_tet = _oracle_per_tet(oracle, w, rng)
    n_s = int(min(max(0.6 * seconds / max(per_tet, 1e-6), 32), w.T))

    def timed(ids, clip, nthreads):
        t0 = time.perf_counter()
        r = oracle.rpd_workload(w, tet_ids=ids, clip=clip, nthreads=nthreads)
        return time.perf_counter() - t0, r

    # deterministic subset (BASELINE.md CPU-baseline plan): every k-th block of 1024
    # consecutive tets -- the tets are in Morton order of their centroids (rpd_workloads), so a
    # block is a compact patch of the mesh -- with k set by the time budget
    blk = 1024
    n_blk = -(-w.T // blk)
    stride = max(1, -(-n_blk * blk // max(n_s, 1)))
    ids = np.concatenate([np.arange(b * blk, min((b + 1) * blk, w.T))
                          for b in range(0, n_blk, stride)]).astype(np.int32)
    n_s = len(ids)
    t_full, r = timed(ids, True, cores)
    t_filt, _ = timed(ids, False, cores)
    n_cand = len(r["cand_idx"])
    # one thread: a sample about cores x smaller (same per-tet work)
    n_1 = max(8, n_s // max(cores, 1))
    ids1 = ids[:: max(1, n_s // n_1)][:n_1]
    t1_full, r1 = timed(ids1, True, 1)
    t1_filt, _ = timed(ids1, False, 1)
    t_clip = max(t_full - t_filt, 1e-9)
    t1_clip = max(t1_full - t1_filt, 1e-9)
    st = r["stats"]
    return {"value": n_cand / t_full, "unit": "pairs/s", "cores": cores, "kind": "oracle",
            "cpu": cpu_model(),
            "sample": f"{n_s} tets of {w.T} ({n_s / w.T:.2%}: every {stride}-th Morton block of "
                      f"{blk} tets; full RPD of the {w.N}-sphere set: Alg. 1 over all {w.N} "
                      f"spheres + clip), {t_full:.1f} s; partial updates not sampled",
            "all_cores": {"threads": cores, "tets": int(n_s), "pairs_filtered_per_s":
                          n_s * w.N / t_filt, "pairs_clipped_per_s": n_cand / t_clip,
                          "filter_s": t_filt, "clip_s": t_clip, "full_s": t_full},
            "one_thread": {"threads": 1, "tets": int(len(ids1)), "pairs_filtered_per_s":
                           len(ids1) * w.N / t1_filt,
                           "pairs_clipped_per_s": len(r1["cand_idx"]) / t1_clip,
                           "filter_s": t1_filt, "clip_s": t1_clip, "full_s": t1_full},
            "oracle_counters": {k: int(st[k]) for k in ("n_rel_tests", "n_clip_tests",
                                                         "n_constructions", "n_fan_triangles")}}


# ----------------------------------------------------------------------------- our arm


def load_oracle_work(cfg):
    """Oracle-counted algorithmic work of the bench step (tools/oracle_work.py, committed)."""
    try:
        d = json.load(open(os.path.join(ROOT, "profiles", "oracle_work.json")))
        return d if d.get("config") == cfg else None
    except Exception:
        return None


def ev():
    import torch
    return torch.cuda.Event(enable_timing=True)


def side_euler(args, ctx, w, ids, world, recs, flush, d_verts, d_tets, d_base, to_dev):
    import torch
    import torch.distributed as dist
    import rpd_workloads as W
    dev = d_verts.device
    # ---- NEXT-1 side measurement: the full RPD with the fractional Euler characteristics
    # fused into the clip (payloads from the whole mesh, per-sphere sums all-reduced)
    from paper_2403_18761_b200.dist import allreduce_euler
    L = ctx.set_euler(w.tets, len(w.verts), ids if world > 1 else None)
    e_full, e_clip = [], []
    for s in range(args.warmup + args.steps):
        flush.zero_()
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        ev0.record()
        ctx.relations(d_verts, d_tets, *d_base)
        ctx.clip()
        ev1.record()
        torch.cuda.synchronize()
        if s >= args.warmup:
            st = ctx.stats()
            e_full.append(ev0.elapsed_time(ev1))
            e_clip.append(st["clip_ms"])
    cc_ms = None
    if world == 1:  # CC numbers (NEXT-2) need the whole mesh in one ctx
        cc = []
        for s in range(args.warmup + args.steps):
            ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            ev0.record()
            ctx.topology()
            ev1.record()
            torch.cuda.synchronize()
            if s >= args.warmup:
                cc.append(ev0.elapsed_time(ev1))
        cc_ms = float(np.median(cc))
        topo = ctx.download_topology()
        rp = []
        for s in range(args.warmup + args.steps):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            rpe = ctx.rpe(device=True)
            torch.cuda.synchronize()
            if s >= args.warmup:
                rp.append(1e3 * (time.perf_counter() - t0))
        mm = []
        for s in range(args.warmup + args.steps):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            med = ctx.medial_mesh(device=True)
            torch.cuda.synchronize()
            if s >= args.warmup:
                mm.append(1e3 * (time.perf_counter() - t0))
        # NEXT-4: envelope distance of 100k boundary samples to that medial mesh
        smp = to_dev(W.boundary_samples(w.verts, w.tets, 100_000, seed=5))
        env = []
        for s in range(args.warmup + args.steps):
            ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            ev0.record()
            _, _, n_eval = ctx.envelope(smp, d_base[0], med["edges"], med["faces"],
                                        device=True)
            ev1.record()
            torch.cuda.synchronize()
            if s >= args.warmup:
                env.append(ev0.elapsed_time(ev1))
        n_prims = w.N + int(med["edges"].shape[0]) + int(med["faces"].shape[0])
    eu = ctx.download_euler(device=True)
    if world > 1:
        eu = allreduce_euler(eu, ctx)
    chi = eu["rpc_sum"].cpu().numpy()
    integral = bool(torch.all(eu["rpc_exact"] == 1).item())
    ctx.set_euler(None, 0)
    ef = torch.tensor([float(np.median(e_full)), float(np.median(e_clip))],
                      dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(ef, op=dist.ReduceOp.MAX)
    euler = {"full_rpd_ms": float(ef[0]), "clip_ms": float(ef[1]),
             "clip_overhead_vs_plain": float(ef[1]) / max(float(np.median(
                 [r["clip_ms"] for r in recs])), 1e-9) - 1.0,
             "n_primes": int(L), "rpc_sums_integral": integral,
             "spheres_with_cells": int(np.sum(chi != 0)),
             "rpc_euler_eq_1": int(np.sum(chi == 1)),
             "cc_ms": cc_ms,
             "rpc_cc_eq_1": int(np.sum(topo["rpc_cc"] == 1)) if cc_ms is not None else None,
             "rpc_cc_gt_1": int(np.sum(topo["rpc_cc"] > 1)) if cc_ms is not None else None,
             "medial_mesh_ms": float(np.median(mm)) if cc_ms is not None else None,
             "rpe_ms": float(np.median(rp)) if cc_ms is not None else None,
             "rpe_triples": int(rpe["tri"].shape[0]) if cc_ms is not None else None,
             "rpe_euler_eq_1": int(((rpe["tri_euler"] // rpe["euler_denom"]) == 1).sum().item())
             if cc_ms is not None else None,
             "rpe_cc_eq_1": int((rpe["tri_cc"] == 1).sum().item())
             if cc_ms is not None else None,
             "medial_edges": int(med["edges"].shape[0]) if cc_ms is not None else None,
             "medial_faces": int(med["faces"].shape[0]) if cc_ms is not None else None,
             "envelope": {"samples": 100_000, "primitives": n_prims,
                          "ms": float(np.median(env)), "pairs_evaluated": int(n_eval),
                          "pairs_total": 100_000 * n_prims,
                          "note": "NEXT-4 envelope distance (PAPER.md:520-542): boundary "
                                  "samples vs the medial mesh's spheres/cones/slabs, "
                                  "closed forms with exact tile culling"}
             if cc_ms is not None else None,
             "note": "fractional Euler characteristics (PAPER.md:482-506) fused into the "
                     "clip; full_rpd_ms = relations + clip + per-sphere sums (CUDA events); "
                     "cc_ms = CC numbers of all RPCs / RPFs (PAPER.md:461-466, union-find); "
                     "medial_mesh_ms = dual medial mesh extraction (host-timed, two syncs)"}
    return euler


def side_neighbors(args, ctx, w, flush, d_verts, d_tets, d_base):
    import torch
    import rpd_workloads as W
    # ---- NEXT-3 side measurement: the sphere neighbour lists on the GPU, the
    # step before the RPD (an input in the timed step); then the full RPD with those lists
    box = W.mesh_box(w.verts)
    nb_ms = []
    for s in range(args.warmup + args.steps):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        g = ctx.neighbors(d_base[0], box, device=True)
        torch.cuda.synchronize()
        if s >= args.warmup:
            nb_ms.append(1e3 * (time.perf_counter() - t0))

    def full_rpd(off, idx):
        ms = []
        for s in range(2):
            flush.zero_()
            torch.cuda.synchronize()
            ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            ev0.record()
            ctx.relations(d_verts, d_tets, d_base[0], off, idx)
            c = ctx.clip()
            ev1.record()
            torch.cuda.synchronize()
            ms.append(ev0.elapsed_time(ev1))
        return ms[-1], c.n_pieces, c.n_inc

    t_gpu, np_gpu, ni_gpu = full_rpd(g["nbr_off"], g["nbr_idx"])
    t_rt, np_rt, ni_rt = full_rpd(d_base[1], d_base[2])
    # incremental lists along the C4 batches (rpd_neighbors_update: only the rows a batch can
    # change are recomputed; reading R34)
    inc_ms, inc_rows = [], []
    if w.batches:
        dev = d_verts.device
        ctx.neighbors(d_base[0], box, device=True)
        n_prev = w.N
        for (sph, _, _) in w.batches:
            d_sph = torch.as_tensor(np.ascontiguousarray(sph)).to(dev)
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            u = ctx.neighbors_update(d_sph, len(sph) - n_prev, box, device=True)
            torch.cuda.synchronize()
            inc_ms.append(1e3 * (time.perf_counter() - t0))
            inc_rows.append(int(u["n_rows"]))
            n_prev = len(sph)
    nbr = {"ms": float(np.median(nb_ms)), "E": int(g["nbr_idx"].numel()),
           "update_ms_per_batch": float(np.median(inc_ms)) if inc_ms else None,
           "update_rows_per_batch": float(np.median(inc_rows)) if inc_rows else None,
           "E_regular_triangulation": int(len(w.nbr_idx)),
           "hidden": int(g["n_hidden"]), "vertex_overflow": int(g["n_vertex_overflow"]),
           "full_rpd_ms_gpu_lists": float(t_gpu), "full_rpd_ms_rt_lists": float(t_rt),
           "pieces_equal_counts": bool(np_gpu == np_rt and ni_gpu == ni_rt),
           "note": "NEXT-3 rpd_neighbors (host-timed around the call, two syncs): certified "
                   "superset of the mesh-box power-cell neighbours; full RPD = relations + "
                   "clip (CUDA events, L2 flushed) with the GPU lists vs the Qhull lists; "
                   "update_*: rpd_neighbors_update after each C4 batch (host-timed), median "
                   "time and rows recomputed"}
    return nbr


def side_small_m(args, ctx, w, d_verts, d_tets, to_dev):
    import torch
    import rpd_workloads as W
    # ---- the paper's regime of few insertions per iteration ("also report
    # M = 1 and M = 10 per-iteration latency"; "few (even single) spheres"): the
    # same C3 start, batches of M = 1 and M = 10 spheres, per-update device time
    small = {}
    t_, n_, mode_, _, _ = W.CONFIGS["C3"]
    for M in (1, 10):
        ws = W.make_shape_workload(f"C4m{M}", t_, n_, seed=args.seed, radius_mode=mode_,
                                   n_batches=6, batch_m=M, clusters=min(M, 10))
        ctx.relations(d_verts, d_tets, to_dev(ws.spheres), to_dev(ws.nbr_off),
                      to_dev(ws.nbr_idx))
        ctx.clip()
        n_prev, lat, nb_lat = ws.N, [], []
        box = W.mesh_box(ws.verts)
        ctx.neighbors(to_dev(ws.spheres), box, device=True)
        for b, (sph, off, idx) in enumerate(ws.batches):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            u = ctx.neighbors_update(to_dev(sph), len(sph) - n_prev, box, device=True)
            torch.cuda.synchronize()
            if b > 0:
                nb_lat.append((1e3 * (time.perf_counter() - t0), int(u["n_rows"])))
            args_b = (to_dev(sph), to_dev(off), to_dev(idx),
                      to_dev(np.arange(n_prev, len(sph), dtype=np.int32)))
            n_prev = len(sph)
            torch.cuda.synchronize()
            ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            ev0.record()
            _, nd = ctx.update_partial(*args_b)
            ev1.record()
            torch.cuda.synchronize()
            if b > 0:   # the first update warms the new shapes up
                lat.append((ev0.elapsed_time(ev1), nd))
        small[f"M{M}"] = {"partial_ms": float(np.median([x[0] for x in lat])),
                          "dirty_tets": float(np.median([x[1] for x in lat])),
                          "updates": len(lat),
                          "neighbors_update_ms": float(np.median([x[0] for x in nb_lat])),
                          "neighbors_rows": float(np.median([x[1] for x in nb_lat]))}
    return small


def main():
    args = parse()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        # N ranks of this script, one per GPU, through torch.distributed.run (127.0.0.1)
        from paper_2403_18761_b200.dist import launch_ranks
        sys.exit(launch_ranks(args.gpus, os.path.abspath(__file__), sys.argv[1:]))
    if args.impl == "reference":
        run_reference(args)
        return
    import torch
    import torch.distributed as dist

    import paper_2403_18761_b200 as P
    import rpd_workloads as W
    from paper_2403_18761_b200.dist import ShardedRPD

    world, rank, local = dist_env()
    # the sharded path (process group, exchanges) whenever several ranks run, or on request
    sharded = world > 1 or (args.force_shard and "WORLD_SIZE" in os.environ)
    if sharded:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if rank == 0:
        P.build()
    if sharded:
        dist.barrier()

    w = W.make_config(args.config, seed=args.seed)
    batches = w.batches if args.partial_iters < 0 else w.batches[:args.partial_iters]
    ctx = P.RPDContext(local, filter_mode=args.filter)
    # the timed steps run without the library's timers (the update graphs' %globaltimer stamps
    # are kernel nodes); the per-step breakdown comes from extra timed-by-the-library steps
    # after the timed region
    ctx.set_profile(False)
    S = ShardedRPD(ctx, w.T) if sharded else None
    ids = S.ids if S else np.arange(w.T, dtype=np.int32)
    tets_local = w.tets[ids]
    to_dev = lambda a: torch.as_tensor(np.ascontiguousarray(a)).to(dev)
    d_verts, d_tets = to_dev(w.verts), to_dev(tets_local)
    d_base = [to_dev(w.spheres), to_dev(w.nbr_off), to_dev(w.nbr_idx)]
    d_batches = []
    n_prev = w.N
    for (sph, off, idx) in batches:
        d_batches.append((to_dev(sph), to_dev(off), to_dev(idx),
                          to_dev(np.arange(n_prev, len(sph), dtype=np.int32))))
        n_prev = len(sph)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)   # > 126 MB L2
    CNT = ("rel_tests", "clip_plane_evals", "clip_vertex_tests", "clip_constructions",
           "clip_fan_triangles", "pairs_clipped", "pairs_filtered", "pairs_tested")

    def step(record):
        """One pass of the hot path: full RPD (+ gather), then the partial updates (+ the
        dirty-segment exchanges).  CUDA events on the ctx's (legacy default) stream."""
        e = [ev() for _ in range(3)]
        e[0].record()
        nc = ctx.relations(d_verts, d_tets, *d_base)
        ctx.clip()
        e[1].record()
        st = ctx.stats_struct()  # (ctypes copy; turned into dicts after the timed region)
        if S:
            S.gather_full()
        e[2].record()
        rec = {"n_cand": nc, "n_pieces": ctx.counts.n_pieces, "st": st, "ev": e,
               "bytes": S.bytes_sent if S else 0, "partial": []}
        for (sph, off, idx, new) in d_batches:
            pe = [ev() for _ in range(3)]
            pe[0].record()
            counts, nd = ctx.update_partial(sph, off, idx, new)
            pe[1].record()
            st = ctx.stats_struct()
            if S:
                S.exchange_partial(nd)
            pe[2].record()
            rec["partial"].append({"n_dirty": nd, "ev": pe, "st": st,
                                   "bytes": S.bytes_sent if S else 0})
        record.append(rec)

    def unpack(recs):
        """ctypes stats -> the fields used below (after the timed region)."""
        for r in recs:
            for d in [r] + r["partial"]:
                st = d.pop("st")
                d["filter_ms"], d["clip_ms"] = st.filter_ms, st.clip_ms
                d["counters"] = {k: getattr(st, k) for k in CNT}

    for s in range(args.warmup):
        step([])
    torch.cuda.synchronize()
    sampler = ClockSampler(local)
    sampler.start()
    st0 = ctx.stats()
    launches0 = st0["kernel_launches"]
    recs, times = [], []
    for s in range(args.steps):
        flush.zero_()
        if sharded:
            dist.barrier()
        torch.cuda.synchronize()
        e0, e1 = ev(), ev()
        e0.record()
        step(recs)
        e1.record()
        torch.cuda.synchronize()
        times.append(e0.elapsed_time(e1))
    st1 = ctx.stats()
    launches = st1["kernel_launches"] - launches0
    # partial updates replayed as CUDA graphs in the timed region (RPD_OPT_GRAPH): replays,
    # captures (one per buffer layout; 0 once warm), eager redos of a batch
    graphs = {k: int(st1["graph_" + k] - st0["graph_" + k])
              for k in ("updates", "captures", "fallbacks")}
    clocks = sampler.stop()
    torch.cuda.synchronize()
    unpack(recs)

    # ---- the same steps with the library's timers on (CUDA events around the full RPD's
    # filter / clip, stamp nodes in the update graphs): the filter / clip split of the
    # breakdown and the clip time of the roofline; outside the timed region
    ctx.set_profile(True)
    step([])  # (captures the stamped update graphs)
    recs_p = []
    for s in range(max(3, min(args.steps, 5))):
        flush.zero_()
        if sharded:
            dist.barrier()
        torch.cuda.synchronize()
        step(recs_p)
        torch.cuda.synchronize()
    unpack(recs_p)
    ctx.set_profile(False)

    def el(p):
        return p[0].elapsed_time(p[1]), p[1].elapsed_time(p[2])

    # pairs clipped: all candidates of the full RPD + the re-clipped pairs of the dirty tets
    pairs_local = sum(r["n_cand"] + sum(p["counters"]["pairs_clipped"] for p in r["partial"])
                      for r in recs)
    t = torch.tensor([float(np.sum(times)), float(pairs_local)], dtype=torch.float64,
                     device=dev)
    if sharded:
        tm = t[:1].clone()
        dist.all_reduce(tm, op=dist.ReduceOp.MAX)
        dist.all_reduce(t, op=dist.ReduceOp.SUM)
        t[0] = tm[0]
    total_ms, pairs_total = float(t[0]), float(t[1])
    value = pairs_total / (total_ms * 1e-3)

    # ---- per-step breakdown (medians over the timed steps; library CUDA events for the
    # filter / clip kernels, bench events around the calls; "other" = staging, compaction,
    # scans, dirty detection, merge copies, launch gaps and host syncs)
    med = lambda xs: float(np.median(xs)) if len(xs) else None
    full_ms = [el(r["ev"])[0] for r in recs]
    gath_ms = [el(r["ev"])[1] for r in recs]
    fmed, cmed = med([r["filter_ms"] for r in recs_p]), med([r["clip_ms"] for r in recs_p])
    pt = [el(p["ev"]) for r in recs for p in r["partial"]]
    p_tot = med([x[0] for x in pt])
    p_f = med([p["filter_ms"] for r in recs_p for p in r["partial"]])
    p_c = med([p["clip_ms"] for r in recs_p for p in r["partial"]])
    n_part = len(d_batches)
    breakdown = {
        "step_ms": total_ms / args.steps,
        "full": {"total": med(full_ms), "filter": fmed, "clip": cmed,
                 "other": med(full_ms) - fmed - cmed},
        "partial_per_update": {"total": p_tot, "filter": p_f, "clip": p_c,
                               "other": (p_tot - p_f - p_c) if p_tot is not None else None,
                               "updates_per_step": n_part},
        "exchange": {"full_gather_ms": med(gath_ms) if S else 0.0,
                     "partial_exchange_ms": med([x[1] for x in pt]) if S else 0.0,
                     "bytes_per_step": int(np.median([r["bytes"] + sum(p["bytes"] for p in
                                                      r["partial"]) for r in recs]))},
        "note": "totals from the timed steps (library timers off); filter = Alg. 1 kernels "
                "(+ dirty detection in partial updates), clip = the clip tiers, both from "
                "extra steps with the library's timers on after the timed region; other = "
                "staging, compaction, scans, merge, launch gaps, syncs",
    }
    clip_step_ms = float(np.median([r["clip_ms"] + sum(p["clip_ms"] for p in r["partial"])
                                    for r in recs_p]))

    # ---- e2e: the same step through the public API with HOST (pinned) buffers: every input
    # array is copied host->device by the library inside the timed region, the exchanges run
    # (N > 1), and the final global piece set is downloaded to pinned host arrays
    pin = lambda a: torch.as_tensor(np.ascontiguousarray(a)).pin_memory().numpy()
    h_in = [pin(w.verts), pin(tets_local), pin(w.spheres), pin(w.nbr_off), pin(w.nbr_idx)]
    h_batches = []
    n_prev = w.N
    for (sph, off, idx) in batches:
        h_batches.append((pin(sph), pin(off), pin(idx),
                          pin(np.arange(n_prev, len(sph), dtype=np.int32))))
        n_prev = len(sph)
    h2d = sum(a.nbytes for a in h_in) + sum(a.nbytes for hb in h_batches for a in hb)
    e2e_times, d2h, e2e_pairs = [], 0, []
    h_out = None
    for s in range(max(2, min(args.steps, 5)) + 1):
        flush.zero_()
        if sharded:
            dist.barrier()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        pairs = ctx.relations(*h_in)
        ctx.clip()
        if S:
            S.gather_full()
        for hb in h_batches:
            _, nd = ctx.update_partial(*hb)
            pairs += ctx.stats()["pairs_clipped"]
            if S:
                S.exchange_partial(nd)
        if S:   # the global CSR (device tensors) -> pinned host
            out = {k: torch.empty(v.shape, dtype=v.dtype, pin_memory=True).copy_(v)
                   for k, v in S.glob.items() if not k.startswith("cand")}
        else:
            if h_out is None:   # pinned destinations sized once (first, untimed, iteration)
                cnt = ctx.counts
                h_out = {k: torch.empty(n, dtype=dt).pin_memory().numpy() for k, n, dt in [
                    ("piece_off", w.T + 1, torch.int32),
                    ("piece_sphere", cnt.n_pieces, torch.int32),
                    ("piece_vol", cnt.n_pieces, torch.float64),
                    ("piece_m1", 3 * cnt.n_pieces, torch.float64),
                    ("piece_facemask", cnt.n_pieces, torch.uint8),
                    ("inc_off", cnt.n_pieces + 1, torch.int32),
                    ("inc_sphere", cnt.n_inc, torch.int32)]}
            out = ctx.download_pieces(out=h_out)
        torch.cuda.synchronize()
        dt = time.perf_counter() - t0
        if s > 0:
            e2e_times.append(dt)
            e2e_pairs.append(pairs)
        d2h = sum((v.numel() * v.element_size()) if isinstance(v, torch.Tensor) else
                  np.asarray(v).nbytes for v in out.values())
    et = torch.tensor([float(np.sum(e2e_times)), float(np.sum(e2e_pairs))],
                      dtype=torch.float64, device=dev)
    if sharded:
        etm = et[:1].clone()
        dist.all_reduce(etm, op=dist.ReduceOp.MAX)
        dist.all_reduce(et, op=dist.ReduceOp.SUM)
        et[0] = etm[0]
    e2e_value = float(et[1]) / float(et[0])

    ctx.set_profile(True)  # (the side records read the library's timers)
    euler = side_euler(args, ctx, w, ids, world if not sharded else max(world, 2), recs_p, flush,
                       d_verts, d_tets, d_base, to_dev) \
        if not args.no_euler else None
    nbr = side_neighbors(args, ctx, w, flush, d_verts, d_tets, d_base) \
        if not args.no_nbr else None
    small = side_small_m(args, ctx, w, d_verts, d_tets, to_dev) \
        if world == 1 and args.config == "C4" and not args.no_small else None

    # ---- roofline of the dominant kernel: the clip (all tiers, full + partial updates of the
    # step) against the FP64 peak; algorithmic flops counted by the ORACLE on the same input
    # (tools/oracle_work.py -> profiles/oracle_work.json) when present
    peak, peak_src = fp64_peak_tflops()
    ow = load_oracle_work(args.config) \
        if len(d_batches) == len(w.batches) and args.seed == 0 else None
    kc = {k: int(np.median([r["counters"][k] + sum(p["counters"][k] for p in r["partial"])
                            for r in recs])) for k in CNT}
    kernel_flops = (24 * kc["clip_plane_evals"] + 8 * kc["clip_vertex_tests"] +
                    40 * kc["clip_constructions"] + 30 * kc["clip_fan_triangles"])
    if ow and world == 1:
        flops = float(ow["full"]["clip_flops"] + ow["partial_total"]["clip_flops"])
        per_unit = ("oracle-counted (profiles/oracle_work.json): 6 flop per vertex-plane test + "
                    "40 per vertex construction + 30 per fan triangle (SURVEY.md §8(d)), C3 full "
                    "RPD + the dirty-tet re-clips of the 10 partial updates")
    else:
        flops = float(kernel_flops) * world
        per_unit = ("kernel-counted: 24 flop per (pair, plane) corner classification + 8 per "
                    "vertex sign test + 40 per vertex construction + 30 per fan triangle")
    achieved = flops / (clip_step_ms * 1e-3) / 1e12 / world
    traffic, ncu = None, None
    try:
        ncu = json.load(open(NCU_TRAFFIC)).get("clip")
        if isinstance(ncu, dict) and ncu.get("config", args.config) != args.config:
            ncu = None  # (the committed capture is of another workload)
        traffic = ncu.get("traffic") if isinstance(ncu, dict) else None
    except Exception:
        pass
    roofline = {"bound": "alu", "achieved": achieved, "peak": peak, "unit": "TFLOP/s",
                "frac": achieved / peak, "traffic": traffic,
                "kernel": "k_clip (all tiers, full RPD + partial updates of the step)",
                "kernel_ms_per_step": clip_step_ms, "algorithmic_flops_per_step": flops,
                "kernel_counted_flops_per_step": float(kernel_flops), "per_unit": per_unit,
                "peak_source": peak_src + "; FP64 DFMA pipe (fp64 ALU bound, no tensor cores)"}
    if isinstance(ncu, dict):
        roofline["ncu"] = {k: ncu[k] for k in ("ipc", "issue_frac", "fp64_pipe_frac",
                                               "warps_active_frac", "lanes_active", "note")
                           if k in ncu}

    line = {
        "metric": "tet-sphere pairs clipped/s",
        "value": value, "unit": "pairs/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": total_ms / args.steps, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic",
        "config": bench_config(args, w, world),
        "full_rpd_ms": breakdown["full"]["total"], "filter_ms": fmed, "clip_ms": cmed,
        "pairs_filtered_per_s": float(recs[0]["counters"]["pairs_filtered"]) * world /
        (fmed * 1e-3),
        "pairs_clipped_per_s_clip_kernel": recs[0]["n_cand"] * world / (cmed * 1e-3),
        "partial_rpd_ms": p_tot,
        "partial_dirty_tets": med([p["n_dirty"] for r in recs for p in r["partial"]]),
        "step_breakdown_ms": breakdown,
        "counters_per_step": kc,
        "roofline": roofline,
        "clocks": clocks,
        "e2e": {"value": e2e_value, "unit": "pairs/s", "h2d_bytes_per_step": int(h2d),
                "d2h_bytes_per_step": int(d2h),
                "note": "the bench step (full RPD + partial updates, + exchanges at N > 1) "
                        "through the C ABI with pinned host inputs and a pinned host download "
                        "of the final global pieces; host-timed, max over ranks"},
        "euler": euler,
        "partial_small_m": small,
        "neighbors": nbr,
        "gpu_launches": int(launches),
        "gpu_launches_per_step": int(launches // max(args.steps, 1)),
        "graph_updates": graphs,
    }
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline(w, args.cpu_seconds)
    if rank == 0:
        print(json.dumps(line), flush=True)
    ctx.close()
    if sharded:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
