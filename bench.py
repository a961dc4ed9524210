#!/usr/bin/env python
"""bench.py -- SpQR decode path on B200: effective HBM GB/s and us/layer on
LLaMA-65B layer shapes, against the roofline, a dense fp16 GEMV, and the
reference's CPU path.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

Workload (BASELINE.json configs[2], LLaMA-65B layer shapes): one decoder
block's seven linear layers -- q,k,v,o 8192x8192, gate,up 22016x8192 and down
8192x22016 -- each a 3-bit SpQR layer (beta1 = beta2 = 16, 3-bit statistics,
1% CSR outliers), batch-1 matvec with fp16 x.  A step = one pass over the
seven layers.  Synthetic data: uniform-random codes with plausible binary16
statistics (bytes are identical to real layers).

Metric: effective GB/s = algorithmic bytes / time, algorithmic bytes per layer
= stream_payload_bytes (layout.hpp:47-64, the compressed layer) + 2n (fp16 x)
+ 4m (fp32 y).  The block's weights are 400 MB (> 126 MB L2), so every step
re-reads them from HBM (no flush needed).

N > 1 (torchrun): each rank holds a 1/N row band of every layer (the
row-sharded wrapper); the all-gather of y is fused into the band kernels (P2P
stores into every rank's y over CUDA IPC / NVLink + a per-rank round counter,
one 32-thread wait launch per group).  The NCCL all-gather path the north star
names is timed beside it ("multi_gpu.nccl_baseline").  value is the whole-job
bytes / max-over-ranks time ("scaling": "strong").
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

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "SpQR matvec µs/layer & HBM GB/s vs roofline (LLaMA shapes) vs fp16 GEMV"
LAYERS = [("q_proj", 8192, 8192), ("k_proj", 8192, 8192), ("v_proj", 8192, 8192),
          ("o_proj", 8192, 8192), ("gate_proj", 22016, 8192), ("up_proj", 22016, 8192),
          ("down_proj", 8192, 22016)]
# launch groups of a decoder block: layers sharing their input are stacked
GROUPS = [("qkv", [0, 1, 2]), ("o", [3]), ("gate_up", [4, 5]), ("down", [6])]
BITS, RATE = 3, 0.01
REASONS = {0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap",
           0x8: "hw_slowdown", 0x10: "sync_boost", 0x20: "sw_thermal_slowdown",
           0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown"}


def workload_config(n_gpus: int) -> dict:
    return {
        "workload": "llama65b-block: q,k,v,o 8192x8192; gate,up 22016x8192; down 8192x22016",
        "weight_bits": BITS, "stat_bits": 3, "beta1": 16, "beta2": 16, "outlier_rate": RATE,
        "batch": 1, "x_dtype": "f16", "layers": len(LAYERS),
        "l2": "weights 400 MB per step > 126 MB L2: inputs larger than L2, no flush",
        "launches": "4 per step: q/k/v stacked (fused QKV), o, gate/up stacked, down; x shared within a group",
        "graph": "10 steps per CUDA graph (PDL between all launches inside), replayed; remainder by a 1-step graph",
        "parallelism": f"row-shard x{n_gpus} + all-gather of y fused into the band kernels (NCCL timed as baseline)"
        if n_gpus > 1 else "single GPU",
    }


def _synth():
    """The synthetic-layer generator (paper_2306_03078_b200/synth.py: numpy
    only, no native code), loaded by file path so the reference arm never
    imports the product package."""
    import importlib.util
    spec = importlib.util.spec_from_file_location("spqr_synth", os.path.join(ROOT, "paper_2306_03078_b200", "synth.py"))
    mod = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mod)
    return mod


def make_streams():
    synth = _synth()
    cache = os.environ.get("SPQR_BENCH_CACHE", "/tmp/spqr_bench_streams")
    os.makedirs(cache, exist_ok=True)
    out = []
    for i, (name, m, n) in enumerate(LAYERS):
        path = os.path.join(cache, f"{name}_{m}x{n}_b{BITS}_r{RATE}_s{i}.spqr")
        if os.path.exists(path):
            s = open(path, "rb").read()
        else:
            s = synth.random_stream(m, n, BITS, 3, 3, RATE, seed=100 + i)
            tmp = f"{path}.{os.getpid()}.tmp"  # ranks of one node may generate concurrently
            with open(tmp, "wb") as f:
                f.write(s)
            os.replace(tmp, path)
        out.append(s)
    return out


def loaded_native_libs() -> list:
    """Shared objects of this repo mapped into the process (for the record)."""
    libs = set()
    try:
        with open("/proc/self/maps") as f:
            for line in f:
                p = line.split()[-1] if line.strip() else ""
                if p.endswith(".so") and p.startswith(ROOT):
                    libs.add(os.path.relpath(p, ROOT))
    except OSError:
        pass
    return sorted(libs)


def alg_bytes(payload: int, m: int, n: int, x_bytes: int = 2) -> int:
    return payload + x_bytes * n + 4 * m


class ClockSampler:
    """nvidia-smi sampling of SM clocks and throttle reasons while the GPU works."""

    def __init__(self, device: int):
        self.device = device
        self.samples = []
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.device),
                 "--query-gpu=clocks.sm,clocks.max.sm,clocks_event_reasons.active,utilization.gpu",
                 "--format=csv,noheader,nounits", "-lms", "50"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except OSError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) >= 4:
                try:
                    self.samples.append((float(parts[0]), float(parts[1]), int(parts[2], 16), float(parts[3])))
                except ValueError:
                    pass

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self) -> dict:
        busy = [s for s in self.samples if s[3] > 0 and not (s[2] & 0x1)] or self.samples
        if not busy:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"], "samples": 0}
        reasons = set()
        for s in busy:
            for bit, name in REASONS.items():
                if s[2] & bit and bit != 0x1:
                    reasons.add(name)
        return {"sm_mhz": statistics.median(s[0] for s in busy), "sm_max_mhz": max(s[1] for s in busy),
                "reasons": sorted(reasons), "samples": len(busy)}


def host_cpu() -> dict:
    """The box's host CPU (state the cores the CPU numbers ran on)."""
    model = "unknown"
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    model = line.split(":", 1)[1].strip()
                    break
    except OSError:
        pass
    return {"cpu_model": model, "nproc": os.cpu_count(), "affinity": len(os.sched_getaffinity(0))}


def load_peaks() -> tuple[float, str]:
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(p) as f:
            return float(json.load(f)["hbm_gbs"]), "measured"
    except (OSError, KeyError, ValueError):
        return 6650.0, "fallback"


def cpu_reference_sample(streams) -> dict:
    """The reference's own matvec(t, x, plan) (oracle/_ref, kernel.hpp:89) on
    one pass over the block's seven layers, single thread (the reference is
    single-threaded by construction)."""
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import oracle as O

    ref = O.Reference()
    total_bytes, total_t = 0, 0.0
    for (name, m, n), s in zip(LAYERS, streams):
        t = ref.decode(s)
        x = np.random.default_rng(2).standard_normal(n).astype(np.float16).astype(np.float32)
        t0 = time.perf_counter()
        t.matvec(x)
        total_t += time.perf_counter() - t0
        total_bytes += alg_bytes(len(s) - 48, m, n, 4)
        del t
    return {"value": total_bytes / total_t / 1e9, "unit": "GB/s", "cores": 1, "kind": "reference",
            "sample": "one pass over the 7 layers of the block, reference matvec(t, x, plan), 1 thread",
            "seconds": round(total_t, 3), "host": host_cpu()}


def reference_check(streams, groups, rank: int, world: int) -> dict:
    """Refuse to time a wrong kernel (the reference's own guard, kernel.hpp:
    189-192): one matvec of every launch group on this rank's row band, checked
    member by member against the reference's matvec(t, x, plan) on the same
    fp16 x widened to fp32 -- relative L2 (kernel.hpp:154-163) <= 1e-3, the
    north star's bound.  Exits non-zero otherwise."""
    import torch

    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import oracle as O

    ref = O.Reference()
    threads = max(1, len(os.sched_getaffinity(0)) // max(1, int(os.environ.get("LOCAL_WORLD_SIZE", world))))
    worst = {}
    for gp in groups:
        gp["L"].matvec(gp["x"], gp["y"])
        torch.cuda.synchronize()
        y = gp["y"].cpu().numpy()
        x32 = gp["x"].float().cpu().numpy()
        errs = []
        for i, r0, r1, off in gp["local"]:
            t = ref.decode(streams[i])
            nb = max(1, min(threads, (r1 - r0) // 16))
            edges = [r0 + 16 * (((r1 - r0) // 16) * j // nb) for j in range(nb)] + [r1]
            bands = [ref.slice_rows(t, edges[j], edges[j + 1]) for j in range(nb)]
            del t
            yr = ref.matvec_bands(bands, x32, nb)
            errs.append(O.relative_l2(y[off:off + r1 - r0], yr))
        worst[gp["name"]] = max(errs)
    bad = {k: v for k, v in worst.items() if not v <= 1e-3}
    if bad:
        print(json.dumps({"error": "matvec does not match the reference (relative L2 > 1e-3)", "rank": rank,
                          "relative_l2": worst}), flush=True)
        sys.exit(3)
    return {"max_relative_l2": max(worst.values()), "per_group": worst, "bound": 1e-3,
            "against": "reference matvec(t, x, plan) (oracle/_ref) on this rank's band, same fp16 x"}


# ------------------------------------------------------------ reference arm --
def run_reference(args) -> None:
    """The reference's own CPU implementation of the path (oracle/_ref: the
    unmodified headers compiled by oracle/Makefile) on this box's host cores.
    Never imports or loads the product library: the row bands the thread
    harness runs are cut with the reference's own types (ref_slice_rows)."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import oracle as O

    ref = O.Reference()
    streams = make_streams()
    threads = max(1, len(os.sched_getaffinity(0)))
    bands = []  # per layer: list of reference tensors over row bands
    for (name, m, n), s in zip(LAYERS, streams):
        t = ref.decode(s)
        nb = min(threads, m // 16)
        edges = [16 * ((m // 16) * i // nb) for i in range(nb)] + [m]
        bands.append([ref.slice_rows(t, edges[i], edges[i + 1]) for i in range(nb)])
        del t
    xs = [np.random.default_rng(2).standard_normal(n).astype(np.float16).astype(np.float32) for _, _, n in LAYERS]

    def step(layer_ids):
        for i in layer_ids:
            ref.matvec_bands(bands[i], xs[i], threads)

    t0 = time.perf_counter()
    step(range(len(LAYERS)))
    t_full = time.perf_counter() - t0
    budget = 150.0
    layer_ids = list(range(len(LAYERS)))
    sample = "full block (7 layers) per step"
    if t_full * (args.steps + args.warmup) > budget:  # bound the run: one layer per step
        layer_ids = [0]
        sample = "q_proj 8192x8192 per step (bounded sample)"
    sample_bytes = sum(alg_bytes(len(streams[i]) - 48, LAYERS[i][1], LAYERS[i][2], 4) for i in layer_ids)
    for _ in range(max(0, args.warmup - 1)):
        step(layer_ids)
    t0 = time.perf_counter()
    for _ in range(args.steps):
        step(layer_ids)
    dt = time.perf_counter() - t0
    value = sample_bytes * args.steps / dt / 1e9
    line = {
        "metric": METRIC, "value": round(value, 3), "unit": "GB/s", "impl": "reference",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(1e3 * dt / args.steps, 3), "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": workload_config(args.gpus),
        "cpu_baseline": {"value": round(value, 3), "unit": "GB/s", "cores": threads, "kind": "reference",
                         "sample": f"{sample}; the reference's single-threaded matvec(t, x, plan) (kernel.hpp:89) "
                                   f"run on {threads} row bands by {threads} host threads (oracle/_ref, unmodified "
                                   f"headers; bands cut with the reference's own types, ref_slice_rows)",
                         "host": host_cpu()},
        "e2e": {"value": round(value, 3), "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "native_libs": loaded_native_libs(),
    }
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------ our arm --
def run_ours(args) -> None:
    import torch
    import torch.distributed as dist

    import paper_2306_03078_b200 as P

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    # test hook: SPQR_BENCH_SHARE_GPU=1 runs every rank on cuda:0 over gloo, so
    # the N > 1 code path can be exercised on a one-GPU box (not a bench number)
    share = os.environ.get("SPQR_BENCH_SHARE_GPU") == "1"
    if share:
        local = 0
    if world > 1:
        torch.cuda.set_device(local)
        if share:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    dev = torch.device("cuda", local if world > 1 else 0)
    torch.cuda.set_device(dev)

    streams = make_streams()
    from paper_2306_03078_b200.sharded import gather_rows, row_bands

    # One decoder block as a serving stack runs it: q/k/v share x (one stacked
    # handle = fused QKV), gate/up share x (stacked), o and down alone -> four
    # launches per step over the same seven layers' bytes.  N > 1: the rows of
    # each stacked group are cut into row bands (row_bands over the stacked
    # rows, the edges spqr_sharded_create computes), so the gathered y of a
    # group is in [q; k; v] order.  The band layers come from the C ABI's NCCL
    # sharded handles (spqr_sharded_*: band + ncclAllGather = the NCCL
    # baseline), or -- gloo test hook -- from the same slices made here.
    comm = None
    if world > 1 and not share:
        uid = [P.nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(uid, src=0)
        comm = P.NcclComm(uid[0], world, rank, dev.index)
    groups = []
    bytes_step = 0  # whole-job algorithmic bytes per step
    gen = torch.Generator(device="cpu").manual_seed(2)
    for gname, members in GROUPS:
        n = LAYERS[members[0]][2]
        m_total = sum(LAYERS[i][1] for i in members)
        bands = row_bands(m_total, world)
        a, b = bands[rank]
        local, base = [], 0  # (member, member rows r0..r1 on this rank, offset in the band's y)
        for i in members:
            m = LAYERS[i][1]
            la, lb = max(a, base), min(b, base + m)
            if la < lb:
                local.append((i, la - base, lb - base, la - a))
            base += m
            bytes_step += alg_bytes(len(streams[i]) - 48, m, n) + 2 * n * (world - 1)
        S = None
        if comm is not None:
            S = P.ShardedNccl([streams[i] for i in members], comm, device=dev.index)
            assert S.band == (a, b) and S.rows == m_total
            L = S.band_layer()
        else:
            parts = [streams[i] if (r0, r1) == (0, LAYERS[i][1]) else P.slice_rows(streams[i], r0, r1)
                     for i, r0, r1, _ in local]
            L = P.Layer(parts[0], device=dev.index) if len(parts) == 1 else P.Layer.stacked(parts, device=dev.index)
        assert L.info["fast_path"] == 1 and L.rows == b - a
        x = torch.randn(n, generator=gen).to(torch.float16)
        groups.append({
            "name": gname, "members": members, "local": local, "m": m_total, "n": n, "L": L, "S": S,
            "x": x.to(dev), "x32": x.float().pin_memory(), "y": torch.empty(b - a, device=dev),
            "band": (a, b), "bands": bands,
            "yfull": torch.empty(m_total, device=dev) if world > 1 else None,
        })
    payload_step = sum(len(s) - 48 for s in streams)
    check = reference_check(streams, groups, rank, world)  # before any timing

    stream = torch.cuda.Stream(device=dev)
    fused = world > 1
    if fused:  # the product path: all-gather fused into the band kernels (P2P stores + round counters)
        from paper_2306_03078_b200.sharded import FusedGather
        err = ""
        try:
            for gp in groups:
                gp["fg"] = FusedGather(gp["m"], gp["bands"], rank, world, dev.index)
        except Exception as ex:  # noqa: BLE001 -- every rank must agree before choosing a path
            err = f"{type(ex).__name__}: {ex}"
        ok = torch.tensor([0 if err else 1], device=dev)
        dist.all_reduce(ok, op=dist.ReduceOp.MIN)
        fused = bool(ok.item())
        if not fused and rank == 0:
            print(f"fused all-gather unavailable ({err or 'on another rank'}); timing the NCCL path", file=sys.stderr)

    def gather(gp):  # gloo test hook only (torch.distributed all-gather of the y bands)
        gather_rows(gp["y"], gp["bands"], out=gp["yfull"])

    def nccl_step():  # the baseline the north star names: band kernel, then NCCL all-gather (C ABI)
        for gp in groups:
            if gp["S"] is not None:
                gp["S"].matvec(gp["x"], gp["yfull"], stream=stream)
            else:
                gp["L"].matvec(gp["x"], gp["y"], stream=stream)
                gather(gp)

    def step():
        if world > 1 and not fused:
            nccl_step()
            return
        for gp in groups:
            if fused:
                gp["fg"].matvec(gp["L"], gp["x"], stream=stream)
            else:
                gp["L"].matvec(gp["x"], gp["y"], stream=stream)

    with torch.cuda.stream(stream):
        for _ in range(3):
            step()
    torch.cuda.synchronize()
    # CUDA graphs of SPG steps (a serving stack captures a whole decode pass --
    # every block's launches back to back -- in one graph, so block boundaries
    # inside it overlap through PDL like the launches within a block) and of
    # one step for the remainder; K steps = K // SPG long replays + K % SPG short
    SPG = 10
    graph = graph1 = None
    if world == 1 or fused or not share:  # gloo collectives cannot be captured
        graph, graph1 = torch.cuda.CUDAGraph(), torch.cuda.CUDAGraph()
        with torch.cuda.graph(graph, stream=stream):
            for _ in range(SPG):
                step()
        with torch.cuda.graph(graph1, stream=stream):
            step()
        torch.cuda.synchronize()

    def replay(n):
        with torch.cuda.stream(stream):
            if graph is None:
                for _ in range(n):
                    step()
                return
            for _ in range(n // SPG):
                graph.replay()
            for _ in range(n % SPG):
                graph1.replay()

    # clocks: sample through a ~1.5 s soak plus the timed region
    with ClockSampler(dev.index) as clk:
        t_end = time.time() + 1.5
        while time.time() < t_end:
            replay(50)
            stream.synchronize()
        replay(args.warmup)
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        replay(args.steps)
        e1.record(stream)
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
    ms = e0.elapsed_time(e1)
    if world > 1:
        t = torch.tensor([ms], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    ms_per_step = ms / args.steps
    value = bytes_step / (ms_per_step * 1e-3) / 1e9

    # launches of our kernels per step, counted by the library (one C-ABI call per group)
    launches_per_step = 0
    with torch.cuda.stream(stream):
        for gp in groups:
            if fused:  # one more round on every rank (symmetric): band kernel + wait
                gp["fg"].g.matvec(gp["L"], gp["x"], stream=stream)
                launches_per_step += P.last_launch_count()
                gp["fg"].g.wait(stream=stream)
            else:
                gp["L"].matvec(gp["x"], gp["y"], stream=stream)
            launches_per_step += P.last_launch_count()
    torch.cuda.synchronize()

    # ---- dominant kernel alone (no all-gather), per group and over the block ----
    def graph_time(fn, reps, inner=SPG):
        """ms per fn(): `inner` calls captured back to back in one graph (as
        the step), the graph replayed ceil(reps / inner) times."""
        g = torch.cuda.CUDAGraph()
        with torch.cuda.stream(stream):
            fn()
        torch.cuda.synchronize()
        with torch.cuda.graph(g, stream=stream):
            for _ in range(inner):
                fn()
        with torch.cuda.stream(stream):
            for _ in range(2):
                g.replay()
        torch.cuda.synchronize()
        nrep = max(1, -(-reps // inner))
        a_, b_ = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a_.record(stream)
        with torch.cuda.stream(stream):
            for _ in range(nrep):
                g.replay()
        b_.record(stream)
        torch.cuda.synchronize()
        return a_.elapsed_time(b_) / (nrep * inner)

    kms = graph_time(lambda: [gp["L"].matvec(gp["x"], gp["y"], stream=stream) for gp in groups],
                     max(20, args.steps // 5))
    kbytes = sum(alg_bytes(gp["L"].info["payload_bytes"], gp["L"].rows, gp["n"]) for gp in groups)  # this rank
    peak, peak_kind = load_peaks()
    achieved = kbytes / (kms * 1e-3) / 1e9
    traffic = None  # ncu dram__bytes_read+write per launch, averaged over the block's launches
    tf = os.path.join(ROOT, "profiles", "gemv_traffic.json")
    if os.path.exists(tf) and world == 1:
        try:
            with open(tf) as f:
                traffic = json.load(f).get("dram_bytes_per_launch_avg")
        except (OSError, ValueError):
            traffic = None
    roofline = {"bound": "hbm", "achieved": round(achieved, 1), "peak": peak, "unit": "GB/s",
                "frac": round(achieved / peak, 4), "traffic": traffic, "peak_kind": peak_kind,
                "kernel": "gemv_cta (fused x preparation + decode-GEMV + CSR merge, one launch per group)",
                "us_per_launch": round(1e3 * kms / len(groups), 3),
                "alg_bytes_per_launch": kbytes // len(groups)}

    # ---- per group: us per launch (L2-defeating copies are not needed: every
    # group is >= 33 MB and the four groups cycle through 400 MB) ----
    per_layer = {}
    for gp in groups:
        us = 1e3 * graph_time(lambda gp=gp: gp["L"].matvec(gp["x"], gp["y"], stream=stream), 50)
        pb = gp["L"].info["payload_bytes"]
        per_layer[f"{gp['name']} {gp['L'].rows}x{gp['n']}"] = {
            "us": round(us, 3), "us_per_member_layer": round(us / len(gp["members"]), 3),
            "GB/s": round(alg_bytes(pb, gp["L"].rows, gp["n"]) / (us * 1e-6) / 1e9, 1),
            "l2_resident_risk": pb < 126e6}

    # ---- multi-GPU split: kernels alone, all-gathers alone, the
    # step, each the max over ranks ----
    multi = None
    if world > 1:
        def eager_ms(fn, reps=10):  # gloo collectives cannot be captured: host-timed
            fn()
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            for _ in range(reps):
                fn()
            torch.cuda.synchronize()
            return 1e3 * (time.perf_counter() - t0) / reps
        nms = None
        if not share:
            try:  # NCCL collectives inside a CUDA graph
                nms = graph_time(nccl_step, max(20, args.steps // 5))
            except Exception as ex:  # noqa: BLE001 -- the baseline must not sink the run
                print(f"NCCL graph capture failed ({type(ex).__name__}: {ex}); timing it eagerly", file=sys.stderr)
                torch.cuda.synchronize()
        if nms is None:
            nms = eager_ms(nccl_step)
        t = torch.tensor([kms, nms], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        multi = {"path": "fused all-gather: band gemv_cta stores y rows into every rank's buffer (CUDA IPC / "
                         "NVLink P2P) + round counters, one gather_wait launch per group" if fused
                         else "band gemv_cta + NCCL all-gather (spqr_sharded_matvec; fused path unavailable)",
                 "bands": "row_bands over each group's stacked rows: gathered y in [q; k; v] / [gate; up] order",
                 "kernel_us_per_step": round(1e3 * float(t[0]), 3),
                 "step_us": round(1e3 * ms_per_step, 3),
                 "gather_us_per_step": round(1e3 * ms_per_step - 1e3 * float(t[0]), 3),
                 "nccl_baseline": {"step_us": round(1e3 * float(t[1]), 3),
                                   "allgather_us_per_step": round(1e3 * (float(t[1]) - float(t[0])), 3),
                                   "path": "spqr_sharded_matvec (C ABI: band spqr_matvec + ncclAllGather)"
                                           if not share else "band matvec + torch.distributed gloo all-gather"},
                 "allgathers_per_step": len(groups),
                 "allgather_bytes_per_rank": [4 * (gp["band"][1] - gp["band"][0]) for gp in groups]}

    # ---- dense fp16 GEMV comparator (ours and cuBLAS), same stacked shapes ----
    dense = {}
    if world == 1:
        W16 = [torch.randn(gp["m"], gp["n"], device=dev, dtype=torch.float16) * 0.02 for gp in groups]
        yd = [torch.empty(gp["m"], device=dev) for gp in groups]
        for label, fn in (("ours", lambda i: P.dense_gemv_f16(W16[i], groups[i]["x"], yd[i], groups[i]["m"],
                                                               groups[i]["n"], stream=stream)),
                          ("cublas", lambda i: torch.mv(W16[i], groups[i]["x"]))):
            with torch.cuda.stream(stream):
                for i in range(len(groups)):  # eager warm-up (creates the cuBLAS handle)
                    fn(i)
            torch.cuda.synchronize()
            dense[label] = graph_time(lambda: [fn(i) for i in range(len(groups))], 20)
        best = min(dense.values())
        dense = {"ms_per_step_ours": round(dense["ours"], 4), "ms_per_step_cublas": round(dense["cublas"], 4),
                 "dense_bytes_per_step": sum(2 * gp["m"] * gp["n"] + 2 * gp["n"] + 4 * gp["m"] for gp in groups),
                 "speedup_spqr_vs_best_dense": round(best / ms_per_step, 3),
                 "shapes": "same stacked groups as ours (fused QKV, fused gate/up, o, down)"}
        del W16, yd

    # ---- end to end through the public API with host buffers ----
    e2e_steps = max(5, min(args.steps, 50))
    ys_h = [torch.empty(gp["m"], dtype=torch.float32).pin_memory() for gp in groups]
    xs_np = [gp["x32"].numpy() for gp in groups]  # numpy views of the page-locked buffers, made once
    ys_np = [t.numpy() for t in ys_h]
    xd32 = [torch.empty(gp["n"], device=dev, dtype=torch.float32) for gp in groups]

    # world 1: each group's C-ABI host call bound once to its page-locked x / y
    # (Layer.host_call: the per-call Python argument handling is gone; the C
    # call does the same work as matvec_host)
    host_calls = [gp["L"].host_call(xs_np[i], ys_np[i]) for i, gp in enumerate(groups)] if world == 1 else None

    def e2e_step():
        for i, gp in enumerate(groups):
            if world == 1:  # x and y pinned: the call's copies are plain DMA
                host_calls[i]()
            else:
                xd32[i].copy_(gp["x32"], non_blocking=True)
                if fused:
                    yf = gp["fg"].matvec(gp["L"], xd32[i], stream=torch.cuda.current_stream())
                elif gp["S"] is not None:
                    gp["S"].matvec(xd32[i], gp["yfull"], stream=torch.cuda.current_stream())
                    yf = gp["yfull"]
                else:
                    gp["L"].matvec(xd32[i], gp["y"], stream=torch.cuda.current_stream())
                    gather(gp)
                    yf = gp["yfull"]
                ys_h[i].copy_(yf[: gp["m"]], non_blocking=True)
                torch.cuda.current_stream().synchronize()

    for _ in range(2):
        e2e_step()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    t0 = time.perf_counter()
    for _ in range(e2e_steps):
        e2e_step()
    torch.cuda.synchronize()
    e2e_s = time.perf_counter() - t0
    if world > 1:
        t = torch.tensor([e2e_s], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_s = float(t.item())
    e2e = {"value": round(bytes_step * e2e_steps / e2e_s / 1e9, 3), "unit": "GB/s",
           "h2d_bytes_per_step": sum(4 * gp["n"] for gp in groups),
           "d2h_bytes_per_step": sum(4 * gp["m"] for gp in groups),
           "ms_per_step": round(1e3 * e2e_s / e2e_steps, 3),
           "path": "spqr_matvec_host (C ABI, page-locked host x/y bound once per group via Layer.host_call: copy kernel reads x, fused kernel stores y to host, sync) per group"
                   if world == 1 else ("H2D x, spqr_matvec_gather + spqr_gather_wait (fused all-gather), D2H y per group"
                                       if fused else "H2D x, spqr_sharded_matvec (band + NCCL all-gather), D2H y per group")}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            cpu = cpu_reference_sample(streams)
        except Exception as ex:  # noqa: BLE001 -- reported, never fatal
            cpu = {"value": None, "unit": "GB/s", "cores": 1, "kind": "reference", "sample": f"unavailable: {ex}"}

    if rank == 0:
        line = {
            "metric": METRIC, "value": round(value, 3), "unit": "GB/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms_per_step, 5),
            "us_per_layer": round(1e3 * ms_per_step / len(LAYERS), 3),
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
            "dtype": "f16", "data": "synthetic",
            "config": workload_config(world),
            "bytes_per_step": bytes_step, "payload_bytes_per_step": payload_step,
            "roofline": roofline, "per_layer": per_layer, "dense_fp16": dense or None,
            "cpu_baseline": cpu, "e2e": e2e, "clocks": clk.summary(), "multi_gpu": multi,
            "gpu_launches": args.steps * launches_per_step,
            "parity": check, "native_libs": loaded_native_libs(),
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=500)
    ap.add_argument("--warmup", type=int, default=50)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
