"""Benchmark of the grouped-IVF search path on B200 (BASELINE.json metric:
queries/sec at fixed recall@10; ADC scan GB/s vs HBM).

A step = one pass of the search path (probe -> group scores/prune/budget ->
LUT + ADC scan -> top-k) over one batch of queries.  Default workload =
BASELINE.json configs[1] (N=100M, d=96, K=2^16, L=64, M=16, 10^4 queries,
k=100) on seeded synthetic data built on the GPU (paper_1802_02422_b200.builder).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--workload c2|c1|c3|c4|c3mini|c4mini] [--nprobe P] [--tau T] [--candidates C]

N>1 runs under torchrun.  Default `--layout queries`: every rank holds the
whole index and searches a batch of 10^4 queries per step (the synthetic
query set; queries are independent units: no data-path collective; weak
scaling, value = all ranks' queries / the slowest rank's time).  `--layout lists`: every
rank holds a slice of every inverted list and the per-rank top-k lists are
all-gathered over NCCL and merged by K7 (strong scaling).
`--impl reference` times the CPU oracle port of the reference path on the
host cores (rank 0 only).
"""

from __future__ import annotations

import argparse
import hashlib
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

WORKLOADS = {
    # BASELINE.json configs[1]: the single-B200 configuration
    "c2": dict(n=100_000_000, d=96, n_clusters=65536, k=65536, l=64, m=16, nq=10_000,
               nprobe=64, tau=0.5, candidates=10_000, topk=100, kmeans_iters=8, pq_iters=10,
               n_learn=2_000_000),
    # BASELINE.json configs[0]: the reference's CPU-runnable case
    "c1": dict(n=1_000_000, d=96, n_clusters=4096, k=4096, l=64, m=8, nq=1000,
               nprobe=32, tau=0.5, candidates=10_000, topk=100, kmeans_iters=10, pq_iters=15,
               n_learn=100_000),
    # BASELINE.json configs[2] on one B200 (1B x 96, K = 2^20, M = 16; the
    # 8-GPU layout shards these lists).  Built with TF32 assignments, 8M learn
    # rows and 3 Lloyd iterations so the build fits a session.
    "c3": dict(n=1_000_000_000, d=96, n_clusters=1 << 20, k=1 << 20, l=64, m=16, nq=10_000,
               nprobe=64, tau=0.5, candidates=10_000, topk=100, kmeans_iters=3, pq_iters=8,
               n_learn=8_000_000, fast=True),
    # BASELINE.json configs[3] on one B200: 1B x 128 SIFT-like uint8 rows
    # (builder.SynthSpec kind='sift_u8'), K = 2^20, M = 16
    "c4": dict(n=1_000_000_000, d=128, n_clusters=1 << 20, k=1 << 20, l=64, m=16, nq=10_000,
               nprobe=64, tau=0.5, candidates=10_000, topk=100, kmeans_iters=3, pq_iters=8,
               n_learn=8_000_000, fast=True, kind="sift_u8"),
    "c4mini": dict(n=50_000_000, d=128, n_clusters=1 << 18, k=1 << 18, l=64, m=16, nq=10_000,
                   nprobe=64, tau=0.5, candidates=10_000, topk=100, kmeans_iters=3, pq_iters=8,
                   n_learn=2_000_000, fast=True, kind="sift_u8"),
    # a smaller rehearsal of the c3 build path
    "c3mini": dict(n=50_000_000, d=96, n_clusters=1 << 18, k=1 << 18, l=64, m=16, nq=10_000,
                   nprobe=64, tau=0.5, candidates=10_000, topk=100, kmeans_iters=3, pq_iters=8,
                   n_learn=2_000_000, fast=True),
}


def log(msg):
    print(msg, file=sys.stderr, flush=True)


# ---------------------------------------------------------------- workload


BUILD_KEYS = ("n", "d", "n_clusters", "k", "l", "m", "nq", "kmeans_iters", "pq_iters", "n_learn",
              "fast", "kind")


def workload_key(w, noise, seed):
    """Cache key over the fields that shape the index (not the search params)."""
    b = {k_: w[k_] for k_ in BUILD_KEYS if k_ in w}
    s = json.dumps({**b, "noise": noise, "seed": seed, "v": 4}, sort_keys=True)
    return hashlib.blake2b(s.encode(), digest_size=8).hexdigest()


def param_sweep(sx, q_dev, gt, w, k, settings, flush, steps=3):
    """BASELINE configs[1]/[2] nprobe x tau sweeps on the resident index:
    device-timed queries/sec (CUDA events, L2 flushed) and recall@10 per
    (nprobe, tau) at the workload's candidate budget."""
    import torch

    from paper_1802_02422_b200 import SearchParams
    from paper_1802_02422_b200.query import recall_at_r

    out = []
    nq = q_dev.shape[0]
    for nprobe, tau in settings:
        params = SearchParams(nprobe=nprobe, tau=tau, candidates=w["candidates"], ef_search=w["k"])
        for _ in range(2):  # warm-up (workspace sizing, first-use costs)
            ids, _, stats = sx.search_topk(q_dev, params, k)
        torch.cuda.synchronize()
        ms = 0.0
        for _ in range(steps):
            l2_flush(flush)
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            ids, _, stats = sx.search_topk(q_dev, params, k)
            b.record()
            torch.cuda.synchronize()
            ms += a.elapsed_time(b)
        ids_h = ids.cpu().numpy() if hasattr(ids, "cpu") else np.asarray(ids)
        st_h = stats.cpu().numpy() if hasattr(stats, "cpu") else np.asarray(stats)
        out.append({"nprobe": nprobe, "tau": tau, "candidates": w["candidates"],
                    "qps": nq * steps / (ms / 1e3),
                    "recall@10": recall_at_r(list(ids_h), gt, 10),
                    "codes_scanned_mean": float(st_h[:, 3].mean())})
        log(f"[sweep] nprobe={nprobe} tau={tau}: {out[-1]['qps']:.0f} q/s  "
            f"r@10 {out[-1]['recall@10']:.4f}")
    return out


def latency_sweep(dev, queries, w, k, batches=(1, 16, 256, 4096, 10000),
                  budgets=(10_000, 30_000, 100_000), min_queries=20_000, max_calls=400):
    """BASELINE.json configs[4]: per-call latency of search_batch through the
    public API (host queries in pinned memory, host results) at each query
    batch size and candidate budget; p50/p99 over repeated calls, each on a
    different slice of the query set, and queries/sec = batch / mean."""
    import torch

    from paper_1802_02422_b200 import SearchParams
    from paper_1802_02422_b200.query import search_batch

    out = []
    qh = torch.from_numpy(queries).pin_memory().numpy()
    nq = qh.shape[0]
    for cand in budgets:
        params = SearchParams(nprobe=w["nprobe"], tau=w["tau"], candidates=cand, ef_search=w["k"])
        for b in batches:
            b = min(b, nq)
            calls = int(max(5, min(max_calls, min_queries // b)))
            oi = torch.empty((b, k), dtype=torch.int32).pin_memory().numpy()
            od = torch.empty((b, k), dtype=torch.float32).pin_memory().numpy()
            os_ = torch.empty((b, 4), dtype=torch.int64).pin_memory().numpy()
            for i in range(3):  # warm-up (workspace sizing)
                search_batch(dev, qh[:b], params, k=k, out=(oi, od, os_))
            lat = []
            for i in range(calls):
                s0 = (i * b) % max(1, nq - b + 1)
                q = qh[s0:s0 + b]
                torch.cuda.synchronize()
                t0 = time.perf_counter()
                search_batch(dev, q, params, k=k, out=(oi, od, os_))
                lat.append((time.perf_counter() - t0) * 1e3)
            lat = np.array(lat)
            out.append({"batch": b, "candidates": cand, "calls": calls,
                        "p50_ms": float(np.percentile(lat, 50)),
                        "p99_ms": float(np.percentile(lat, 99)),
                        "qps": float(b / (lat.mean() / 1e3))})
            log(f"[sweep] cand={cand} batch={b}: p50 {out[-1]['p50_ms']:.3f} ms "
                f"p99 {out[-1]['p99_ms']:.3f} ms  {out[-1]['qps']:.0f} q/s")
    return out


def load_or_build(w, noise, seed, device, allow_build=True):
    """Index arrays + queries + ground truth.  Built on the GPU; cached under
    /tmp (a speed-up only -- nothing depends on the cache being present)."""
    from paper_1802_02422_b200.builder import BuildSpec, SynthSpec, build_synthetic
    from paper_1802_02422_b200.device_index import IndexArrays

    cache_dir = os.environ.get("GIVF_BENCH_CACHE", "/tmp/givf_bench_cache")
    path = os.path.join(cache_dir, workload_key(w, noise, seed) + ".npz")
    if os.path.exists(path):
        try:
            z = np.load(path)
            arr = IndexArrays(
                centroids=z["centroids"], alphas=z["alphas"], neighbor_ids=z["neighbor_ids"],
                norm_terms=z["norm_terms"], group_sizes=z["group_sizes"],
                region_offsets=z["region_offsets"], point_ids=z["point_ids"], codes=z["codes"],
                const_bytes=z["const_bytes"], codewords=z["codewords"], rotation=None,
                const_lo=float(z["const_lohi"][0]), const_hi=float(z["const_lohi"][1]),
                grouping=True)
            log(f"[bench] loaded cached workload {path}")
            return arr, z["queries"], z["gt"], 0.0
        except Exception as e:  # noqa: BLE001
            log(f"[bench] cache unreadable ({e}); rebuilding")
    if not allow_build:
        raise RuntimeError("workload cache missing")
    t0 = time.perf_counter()
    data = SynthSpec(d=w["d"], n_clusters=w["n_clusters"], sigma=0.3, noise=noise, seed=seed,
                     kind=w.get("kind", "gauss"))
    spec = BuildSpec(n=w["n"], k=w["k"], l=w["l"], m=w["m"], n_learn=w["n_learn"],
                     kmeans_iters=w["kmeans_iters"], pq_iters=w["pq_iters"], seed=seed,
                     fast=w.get("fast", False))
    arr, queries, gt = build_synthetic(data, spec, w["nq"], gt_t=10, device=device, log=log)
    build_s = time.perf_counter() - t0
    import torch

    torch.cuda.empty_cache()  # the build's temporaries; the index allocates its own
    if (w["n"] > 200_000_000 and not os.environ.get("GIVF_BENCH_CACHE")
            and int(os.environ.get("WORLD_SIZE", "1")) == 1):
        return arr, queries, gt, build_s  # tens of GB: cache only on request
    try:
        os.makedirs(cache_dir, exist_ok=True)
        tmp = path + f".tmp{os.getpid()}.npz"
        np.savez(tmp, centroids=arr.centroids, alphas=arr.alphas, neighbor_ids=arr.neighbor_ids,
                 norm_terms=arr.norm_terms, group_sizes=arr.group_sizes,
                 region_offsets=arr.region_offsets, point_ids=arr.point_ids, codes=arr.codes,
                 const_bytes=arr.const_bytes, codewords=arr.codewords,
                 const_lohi=np.array([arr.const_lo, arr.const_hi]), queries=queries, gt=gt)
        os.replace(tmp, path)
    except OSError as e:
        log(f"[bench] cache write failed: {e}")
    return arr, queries, gt, build_s


# ---------------------------------------------------------------- clocks


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index=0):
        self.gpu = gpu_index
        self.samples = []
        self._stop = threading.Event()
        self._t = None

    def _run(self):
        while not self._stop.is_set():
            try:
                out = subprocess.run(
                    ["nvidia-smi", f"--id={self.gpu}", f"--query-gpu={self.FIELDS}",
                     "--format=csv,noheader,nounits"], capture_output=True, text=True, timeout=5)
                parts = [p.strip() for p in out.stdout.strip().split(",")]
                if len(parts) == 6:
                    self.samples.append(parts)
            except Exception:  # noqa: BLE001
                pass
            self._stop.wait(0.2)

    def __enter__(self):
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()
        return self

    def __exit__(self, *exc):
        self._stop.set()
        if self._t:
            self._t.join(timeout=10)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"], "samples": 0}
        sm = [float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for s in self.samples for i in range(4)
                          if s[2 + i].lower() == "active"})
        return {"sm_mhz": float(np.median(sm)) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "samples": len(self.samples)}


# ---------------------------------------------------------------- CPU arms


def _cpu_worker(args):
    """Oracle port of the reference path on one core over a query slice."""
    arr_path, qi, params, deadline = args
    from threadpoolctl import threadpool_limits

    threadpool_limits(1)  # one BLAS thread per forked worker (no oversubscription)
    from oracle import search_oracle as so

    arr = _CPU_STATE["arr"]
    queries = _CPU_STATE["queries"]
    c = arr.centroids
    c_sq = np.einsum("kd,kd->k", c.astype(np.float64), c.astype(np.float64))
    cmax = float(np.sqrt(c_sq.max()))

    def probe(cc, q, nprobe):
        return so.probe_exact_fast(cc, q, nprobe, c_sq=c_sq, cmax=cmax)

    done = 0
    t0 = time.perf_counter()
    for i in qi:
        if time.perf_counter() > deadline:
            break
        so.search_one(arr, queries[i], params, probe=probe)
        done += 1
    return done, time.perf_counter() - t0


_CPU_STATE = {}


def cpu_port_qps(arr, queries, w, seconds=20.0, cores=None):
    """Time the oracle port (numpy restatement of search.py:93-163 with the
    exact probe) on the host cores: fork one worker per core, each takes a
    strided slice of the queries until the time budget runs out."""
    import multiprocessing as mproc

    from oracle import search_oracle as so

    cores = cores or os.cpu_count() or 1
    _CPU_STATE["arr"] = arr
    _CPU_STATE["queries"] = queries
    p = so.Params(nprobe=w["nprobe"], tau=w["tau"], candidates=w["candidates"])
    os.environ["OPENBLAS_NUM_THREADS"] = "1"
    ctx = mproc.get_context("fork")
    t0 = time.perf_counter()
    deadline = time.time() + seconds
    deadline_pc = time.perf_counter() + seconds
    jobs = [(None, list(range(r, len(queries), cores)), p, deadline_pc) for r in range(cores)]
    with ctx.Pool(cores) as pool:
        res = pool.map(_cpu_worker, jobs)
    wall = time.perf_counter() - t0
    done = sum(r[0] for r in res)
    del deadline
    return done / wall, done, wall, cores


# ---------------------------------------------------------------- GPU arm


def l2_flush(buf):
    buf.add_(1.0)  # writes > L2 (126 MB) between timed steps


def run_ours(args, w):
    import torch

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if world > 1:
        import torch.distributed as dist

        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    from paper_1802_02422_b200 import SearchParams, _native
    from paper_1802_02422_b200.sharded import ShardedIndex

    # rank 0 builds (or loads) the workload; the others load it from the cache
    if rank == 0:
        arr, queries, gt, build_s = load_or_build(w, args.noise, args.seed, f"cuda:{local}")
    if world > 1:
        torch.distributed.barrier()
    if rank != 0:
        arr, queries, gt, build_s = load_or_build(w, args.noise, args.seed, f"cuda:{local}",
                                                  allow_build=False)
    torch.cuda.synchronize()
    # layout: "queries" = every rank holds the whole index and
    # searches its own batch of nq queries per step (queries are independent
    # units: no data-path collective, weak scaling); "lists" = every rank
    # owns a shard of every inverted list, the per-rank top-k lists are
    # all-gathered over NCCL and merged by K7 (the same nq queries for every
    # N: strong scaling)
    lists = args.layout == "lists" and world > 1
    shards = world if lists else 1
    sx = ShardedIndex(arr, rank if lists else 0, shards, device=local)
    params = SearchParams(nprobe=w["nprobe"], tau=w["tau"], candidates=w["candidates"],
                          ef_search=w["k"])
    k = w["topk"]
    q_dev = torch.from_numpy(queries).cuda()
    flush = torch.empty(256 * 1024 * 1024 // 4 * 2, dtype=torch.float32, device="cuda")  # 512 MB
    stream = torch.cuda.current_stream()

    def step():
        return sx.search_topk(q_dev, params, k)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()

    # ---- timed: device-resident queries, CUDA events per step, L2 flushed between
    starts = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    ends = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    launches0 = _native.kernel_launches()
    fb0 = sx.dev.fallback_counts()
    rs0 = sx.dev.plan_fallback_reasons()
    if world > 1:
        torch.distributed.barrier()
    torch.cuda.synchronize()
    with ClockSampler(local) as clocks:
        for i in range(args.steps):
            l2_flush(flush)
            starts[i].record(stream)
            ids, dists, stats = step()
            ends[i].record(stream)
        torch.cuda.synchronize()
    if world > 1:
        torch.distributed.barrier()
    launches = _native.kernel_launches() - launches0
    fb1 = sx.dev.fallback_counts()
    fallbacks = {k_: (fb1[k_] - fb0[k_]) / args.steps for k_ in fb0}
    rs1 = sx.dev.plan_fallback_reasons()
    plan_reasons = {k_: (rs1[k_] - rs0[k_]) / args.steps for k_ in rs0 if rs1[k_] > rs0[k_]}
    step_ms = [s.elapsed_time(e) for s, e in zip(starts, ends)]
    total_ms = float(np.sum(step_ms))
    if world > 1:
        t = torch.tensor([total_ms], device="cuda")
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        total_ms = float(t.item())
    nq = queries.shape[0]
    units = nq * (1 if lists else world)  # queries all ranks searched per step
    qps = units * args.steps / (total_ms / 1e3)
    ids_h = ids.cpu().numpy()
    stats_h = stats.cpu().numpy()
    from paper_1802_02422_b200.query import recall_at_r

    recall = {r: recall_at_r(list(ids_h), gt, r) for r in (1, 10, 100)}

    # ---- per-stage kernel time (separate pass, events on the launching stream)
    # one internal stream here, so each kernel's event-timed duration is its own
    saved_streams = os.environ.get("GIVF_STREAMS")
    os.environ["GIVF_STREAMS"] = "1"
    _native.profile_enable(True)
    _native.profile_read()
    prof_steps = max(1, min(3, args.steps))
    for _ in range(prof_steps):
        l2_flush(flush)
        step()
    torch.cuda.synchronize()
    stages = _native.profile_read()
    _native.profile_enable(False)
    if saved_streams is None:
        os.environ.pop("GIVF_STREAMS", None)
    else:
        os.environ["GIVF_STREAMS"] = saved_streams

    # ---- end to end through the public API with host buffers (pinned)
    from paper_1802_02422_b200.query import search_batch

    e2e_qps = None
    h2d = queries.nbytes
    d2h = nq * k * 8 + nq * 32
    if not lists:  # every rank: its own batch through the public API
        qh = torch.from_numpy(queries).pin_memory().numpy()
        oi = torch.empty((nq, k), dtype=torch.int32).pin_memory().numpy()
        od = torch.empty((nq, k), dtype=torch.float32).pin_memory().numpy()
        os_ = torch.empty((nq, 4), dtype=torch.int64).pin_memory().numpy()
        search_batch(sx.dev, qh, params, k=k, out=(oi, od, os_))
        e2e_t = 0.0
        for _ in range(args.steps):
            l2_flush(flush)
            torch.cuda.synchronize()
            if world > 1:
                torch.distributed.barrier()
            t0 = time.perf_counter()
            search_batch(sx.dev, qh, params, k=k, out=(oi, od, os_))
            e2e_t += time.perf_counter() - t0
        if world > 1:  # slowest rank
            t = torch.tensor([e2e_t], device="cuda")
            torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
            e2e_t = float(t.item())
        e2e_qps = units * args.steps / e2e_t
        assert np.array_equal(oi, ids_h), "e2e results differ from the device-resident run"

    sweep = latency_sweep(sx.dev, queries, w, k) if (args.latency_sweep and world == 1) else None
    psweep = None
    if args.sweep and world == 1:
        settings = [(int(a), float(b)) for a, b in (x.split(":") for x in args.sweep.split(","))]
        psweep = param_sweep(sx, q_dev, gt, w, k, settings, flush)

    if rank != 0:
        return None
    m = w["m"]
    scanned_local = float(stats_h[:, 3].sum()) / shards  # ~ rows this rank scans
    # algorithmic bytes: codes_scanned x (M + 1) per query (M code bytes + the
    # constant byte), summed over the step, over the scan kernels' summed time
    scan_ms, scan_n = stages["scan"]
    scan_ms_step = scan_ms / prof_steps
    scan_bytes = scanned_local * (m + 1)
    scan_gbs = scan_bytes / (scan_ms_step / 1e3) / 1e9 if scan_n else None
    peaks = {}
    try:
        peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:  # noqa: BLE001
        pass
    hbm_peak = float(peaks.get("hbm_gbs", 6650.0))
    traffic = None
    tr_path = os.path.join(ROOT, "profiles", f"ncu_scan_traffic_{args.workload}.json")
    if os.path.exists(tr_path):
        try:
            tr = json.load(open(tr_path))
            # ncu DRAM bytes of one captured scan launch, scaled to this step's
            # queries (same per-query work) so it compares with `achieved`
            traffic = tr["dram_bytes_per_launch"] / tr["queries_per_launch"] * nq / shards
        except Exception:  # noqa: BLE001
            traffic = None
    gemm_ms, gemm_n = stages["probe_gemm"]
    probe_flops = 2.0 * w["k"] * w["d"] * nq
    step_stage_ms = {s: v[0] / prof_steps for s, v in stages.items() if v[1]}
    line = {
        "metric": "queries/sec at fixed recall@10 (synthetic, B200)",
        "value": qps,
        "unit": "queries/s",
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": total_ms / args.steps,
        "higher_is_better": True,
        "scaling": "strong" if args.layout == "lists" else "weak",
        "vs_baseline": None,
        "dtype": "f32/f64 (u8 codes)",
        "data": ("synthetic: seeded SIFT-like uint8 gamma mixture, built on GPU"
                 if w.get("kind") == "sift_u8"
                 else f"synthetic: seeded gaussian mixture, noise={args.noise}, built on GPU"),
        "config": {
            "workload": f"BASELINE configs[{ {'c1': 0, 'c2': 1, 'c4': 3, 'c4mini': 3}.get(args.workload, 2)}] ({args.workload})",
            "n": w["n"], "d": w["d"], "K": w["k"], "L": w["l"], "M": w["m"],
            "queries_per_step": units, "queries_per_rank_step": nq,
            "nprobe": w["nprobe"], "tau": w["tau"],
            "candidates": w["candidates"], "k": k, "noise": args.noise,
            "recall@1": recall[1], "recall@10": recall[10], "recall@100": recall[100],
            "codes_scanned_mean": float(stats_h[:, 3].mean()),
            "l2": "flushed between steps (512 MB write); codes also exceed L2",
            "parallelism": (f"list-shard x{world} (NCCL all-gather + K7 merge)" if lists
                            else f"query-parallel x{world} (index replica per GPU, no collective)"
                            if world > 1 else "single GPU"),
        },
        "roofline": {
            "kernel": "scan (K6 ADC scan + top-k)",
            "bound": "hbm",
            "achieved": scan_gbs,
            "peak": hbm_peak,
            "unit": "GB/s",
            "frac": (scan_gbs / hbm_peak) if scan_gbs else None,
            "traffic": traffic,
            "algorithmic_bytes_per_step": scan_bytes,
            "launches_per_step": scan_n / prof_steps,
            "kernel_ms_per_step": scan_ms_step,
            "peak_source": "MEASURED_PEAKS.json hbm_gbs" if peaks else "fallback 6650",
        },
        "roofline_probe": {
            "kernel": "probe_gemm (K1a: bf16x3 tcgen05 GEMM + split kernel); 2*K*d flops per query",
            "achieved_tflops": (probe_flops / (gemm_ms / prof_steps / 1e3) / 1e12) if gemm_n else None,
            "tensor_flops_per_step_bf16x3": probe_flops * 3 * (288 + 32) / 288,
            "unit": "TFLOP/s",
        },
        "stage_ms_per_step": step_stage_ms,
        "gpu_launches": int(launches),
        "fallback_queries_per_step": fallbacks,
        **({"latency_sweep": sweep} if sweep else {}),
        **({"param_sweep": psweep} if psweep else {}),
        "plan_fallback_reasons_per_step": plan_reasons,
        "e2e": {"value": e2e_qps, "unit": "queries/s", "h2d_bytes_per_step": int(h2d),
                "d2h_bytes_per_step": int(d2h)},
        "clocks": clocks.summary(),
        "build_s": build_s,
    }
    if world == 1 and not args.no_cpu_baseline:
        cps, done, wall, cores = cpu_port_qps(arr, queries, w, seconds=args.cpu_seconds)
        line["cpu_baseline"] = {"value": cps, "unit": "queries/s", "cores": cores, "kind": "port",
                                "sample": f"{done} of {nq} queries in {wall:.1f}s "
                                          f"(oracle port, exact probe, fork x{cores})"}
    return line


def run_reference(args, w):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return None
    import torch

    arr, queries, gt, _ = load_or_build(w, args.noise, args.seed, "cuda:0")
    del torch
    per_step = []
    total_done = 0
    cores = os.cpu_count() or 1
    secs = max(2.0, args.cpu_seconds / max(args.steps + args.warmup, 1))
    for i in range(args.warmup + args.steps):
        qps, done, wall, cores = cpu_port_qps(arr, queries, w, seconds=secs, cores=cores)
        if i >= args.warmup:
            per_step.append(qps)
            total_done += done
    v = float(np.mean(per_step))
    return {
        "impl": "reference",
        "metric": "queries/sec at fixed recall@10 (synthetic, B200)",
        "value": v, "unit": "queries/s", "n_gpus": int(os.environ.get("WORLD_SIZE", "1")),
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * w["nq"] / v,
        "higher_is_better": True, "scaling": "strong" if args.layout == "lists" else "weak",
        "vs_baseline": None,
        "dtype": "f32/f64 (u8 codes)", "data": f"synthetic, noise={args.noise}",
        "config": {"workload": args.workload, "nprobe": w["nprobe"], "tau": w["tau"],
                   "candidates": w["candidates"], "k": w["topk"]},
        "cpu_baseline": {"value": v, "unit": "queries/s", "cores": cores, "kind": "port",
                         "sample": f"{total_done} queries over {args.steps} steps of {secs:.1f}s"},
        "e2e": {"value": v, "unit": "queries/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="c2", choices=sorted(WORKLOADS))
    ap.add_argument("--latency-sweep", action="store_true",
                    help="add BASELINE configs[4]'s batch x budget latency sweep (N=1)")
    ap.add_argument("--sweep", default="",
                    help="extra nprobe:tau settings on the same index, e.g. 32:0.5,128:0.25 (N=1)")
    ap.add_argument("--noise", default="per_coord", choices=["per_coord", "total"])
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--nprobe", type=int)
    ap.add_argument("--tau", type=float)
    ap.add_argument("--candidates", type=int)
    ap.add_argument("--cpu-seconds", type=float, default=20.0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--layout", default="queries", choices=["queries", "lists"],
                    help="N>1: query-parallel replicas (weak scaling) or list shards "
                         "merged over NCCL (strong scaling)")
    args = ap.parse_args()
    args.warmup = max(3, args.warmup)
    w = dict(WORKLOADS[args.workload])
    for key in ("nprobe", "tau", "candidates"):
        if getattr(args, key) is not None:
            w[key] = getattr(args, key)
    line = run_reference(args, w) if args.impl == "reference" else run_ours(args, w)
    if line is not None:
        print(json.dumps(line), flush=True)


if __name__ == "__main__":
    main()
