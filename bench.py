"""Benchmark of the grouped-IVF search path on B200 (BASELINE.json metric:
queries/sec at fixed recall@10; ADC scan GB/s vs HBM).

A step = one pass of the search path (probe -> group scores/prune/budget ->
LUT + ADC scan -> top-k) over one batch of queries.  Default workload =
BASELINE.json configs[2] at its full size on one B200: N = 1B, d = 96,
K = 2^20, L = 64, M = 16, 10^4 queries, k = 100, the nprobe 32-512 sweep and
(configs[4]) the batch x budget latency sweep on the same index.  The index
is built on the GPU at the start of the run from seeded synthetic data
(paper_1802_02422_b200.builder: fused sm_100a assignment / encode kernels,
exact ground truth).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--workload c3|c3m8|c4|c2|c1|c3mini|c4mini] [--noise total|per_coord]
                    [--nprobe P] [--tau T] [--candidates C]

N>1 runs under torchrun.  Default `--layout lists`: every rank
owns a slice of every inverted list and the per-rank top-k lists are
all-gathered over NCCL and merged by K7 (strong scaling: the same index and
queries for every N).  `--layout queries`: every rank holds a whole replica
and searches its own batch (weak scaling, no data-path collective).
`--impl reference` times the reference's CPU query path (the oracle port of
search.py, all host cores, rank 0 only) on the same workload.
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

_C3 = dict(n=1_000_000_000, d=96, n_clusters=1 << 20, k=1 << 20, l=64, m=16, nq=10_000,
           nprobe=64, tau=0.5, candidates=10_000, topk=100, kmeans_iters=4, pq_iters=8,
           n_learn=8_000_000, config=2,
           sweep="32:0.5,64:0.5,128:0.5,256:0.5,512:0.5,64:0.25,256:0.25,512:0.25",
           latency_sweep=True)
WORKLOADS = {
    # BASELINE.json configs[2] on one B200: 1B x 96, K = 2^20, M = 16 (the
    # 8-GPU layout shards these lists); configs[4]'s latency sweep runs on it
    "c3": _C3,
    # configs[2] with M = 8
    "c3m8": dict(_C3, m=8, latency_sweep=False),
    # BASELINE.json configs[3]: 1B x 128 SIFT-like uint8 rows, K = 2^20, M = 16
    "c4": dict(_C3, d=128, kind="sift_u8", config=3, latency_sweep=False,
               sweep="32:0.5,128:0.5,512:0.5"),
    # BASELINE.json configs[1]: 100M x 96, K = 2^16, M = 16
    "c2": dict(n=100_000_000, d=96, n_clusters=65536, k=65536, l=64, m=16, nq=10_000,
               nprobe=64, tau=0.5, candidates=10_000, topk=100, kmeans_iters=8, pq_iters=10,
               n_learn=2_000_000, config=1,
               sweep="16:0.5,32:0.5,64:0.5,128:0.5,256:0.5,64:0.25,256:0.25"),
    # BASELINE.json configs[0]: the reference's CPU-runnable case
    "c1": dict(n=1_000_000, d=96, n_clusters=4096, k=4096, l=64, m=8, nq=1000,
               nprobe=32, tau=0.5, candidates=10_000, topk=100, kmeans_iters=10, pq_iters=15,
               n_learn=100_000, config=0),
    # smaller rehearsals of the 1B shapes
    "c3mini": dict(_C3, n=50_000_000, n_clusters=1 << 18, k=1 << 18, n_learn=2_000_000,
                   latency_sweep=False, sweep=""),
    # K = 2^20 probe / planner shapes on a 100M-row index (quick iterations)
    "c3k": dict(_C3, n=100_000_000, latency_sweep=False, sweep=""),
    "c4mini": dict(_C3, n=50_000_000, d=128, n_clusters=1 << 18, k=1 << 18, n_learn=2_000_000,
                   kind="sift_u8", config=3, latency_sweep=False, sweep=""),
}


def log(msg):
    print(msg, file=sys.stderr, flush=True)


# ---------------------------------------------------------------- workload


BUILD_KEYS = ("n", "d", "n_clusters", "k", "l", "m", "nq", "kmeans_iters", "pq_iters", "n_learn",
              "fast", "kind")


def workload_key(w, noise, seed):
    """Cache key over the fields that shape the index (not the search params)."""
    b = {k_: w[k_] for k_ in BUILD_KEYS if k_ in w}
    s = json.dumps({**b, "noise": noise, "seed": seed, "v": 5}, sort_keys=True)
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
    """Index arrays + queries + ground truth, built on the GPU.  Indexes up
    to 200M rows are cached under /tmp (a speed-up only -- nothing depends on
    the cache being present); larger ones keep their row arrays on the device
    and are rebuilt every run."""
    from paper_1802_02422_b200.builder import BuildSpec, SynthSpec, build_synthetic
    from paper_1802_02422_b200.device_index import IndexArrays

    big = w["n"] > 200_000_000
    cache_dir = os.environ.get("GIVF_BENCH_CACHE", "/tmp/givf_bench_cache")
    path = os.path.join(cache_dir, workload_key(w, noise, seed) + ".npz")
    if not big and os.path.exists(path):
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
                     kmeans_iters=w["kmeans_iters"], pq_iters=w["pq_iters"], seed=seed)
    arr, queries, gt = build_synthetic(data, spec, w["nq"], gt_t=10, device=device, log=log,
                                       rows_on_device=big)
    build_s = time.perf_counter() - t0
    import torch

    torch.cuda.empty_cache()  # the build's temporaries; the index allocates its own
    if big:
        return arr, queries, gt, build_s
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


_CPU_STATE = {}


def _cpu_worker(qi):
    """Oracle port of the reference path (search.py:93-163, exact probe via a
    BLAS shortlist re-checked in float64) on one core over a query slice."""
    from threadpoolctl import threadpool_limits

    threadpool_limits(1)  # one BLAS thread per forked worker (no oversubscription)
    from oracle import search_oracle as so

    st = _CPU_STATE
    arr, queries, params = st["arr"], st["queries"], st["params"]
    c_sq, cmax, gstarts = st["c_sq"], st["cmax"], st["gstarts"]

    def probe(cc, q, nprobe):
        return so.probe_exact_fast(cc, q, nprobe, c_sq=c_sq, cmax=cmax)

    t0 = time.perf_counter()
    for i in qi:
        so.search_one(arr, queries[i], params, probe=probe, gstarts=gstarts)
    return len(qi), time.perf_counter() - t0


class CpuOracle:
    """The reference CPU query path on every host core: one forked worker
    per core (created once), each searching its share of a query sample."""

    def __init__(self, arr, queries, w, cores=None):
        import multiprocessing as mproc

        from oracle import search_oracle as so

        self.cores = cores or os.cpu_count() or 1
        host = arr.to_host() if hasattr(arr, "to_host") else arr
        c64 = host.centroids.astype(np.float64)
        c_sq = np.einsum("kd,kd->k", c64, c64)
        _CPU_STATE.update(
            arr=host, queries=queries,
            params=so.Params(nprobe=w["nprobe"], tau=w["tau"], candidates=w["candidates"]),
            c_sq=c_sq, cmax=float(np.sqrt(c_sq.max())),
            gstarts=so.group_starts(host.group_sizes, host.region_offsets))
        os.environ["OPENBLAS_NUM_THREADS"] = "1"
        self.pool = mproc.get_context("fork").Pool(self.cores)
        self.nq = queries.shape[0]
        self.next = 0

    def run(self, count):
        """Search `count` queries (the next ones in the set); returns
        (queries done, wall seconds)."""
        idx = [(self.next + i) % self.nq for i in range(count)]
        self.next = (self.next + count) % self.nq
        jobs = [idx[r::self.cores] for r in range(self.cores)]
        t0 = time.perf_counter()
        res = self.pool.map(_cpu_worker, jobs)
        return sum(r[0] for r in res), time.perf_counter() - t0

    def rate(self, seconds):
        """Queries/s over about `seconds` of work, in rounds of 4 per core."""
        self.run(self.cores)  # warm-up (imports, page-in of the index)
        done, wall = 0, 0.0
        while wall < seconds:
            d, t = self.run(4 * self.cores)
            done += d
            wall += t
        return done / wall, done, wall

    def close(self):
        self.pool.close()
        self.pool.join()


# ---------------------------------------------------------------- GPU arm


def l2_flush(buf):
    buf.add_(1.0)  # writes > L2 (126 MB) between timed steps


def config_of(args, w, units):
    """The workload description shared by both arms (same keys, same values)."""
    return {
        "workload": f"BASELINE configs[{w['config']}] ({args.workload})",
        "n": w["n"], "d": w["d"], "K": w["k"], "L": w["l"], "M": w["m"],
        "data": w.get("kind", "gauss"), "noise": args.noise if w.get("kind") != "sift_u8" else None,
        "queries_per_step": units, "nprobe": w["nprobe"], "tau": w["tau"],
        "candidates": w["candidates"], "k": w["topk"],
    }


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

    # every rank builds the same index (deterministic seeds); ranks of the
    # lists layout keep only their shard of it
    arr, queries, gt, build_s = load_or_build(w, args.noise, args.seed, f"cuda:{local}")
    torch.cuda.synchronize()
    lists = args.layout == "lists" and world > 1
    shards = world if lists else 1
    sx = ShardedIndex(arr, rank if lists else 0, shards, device=local)
    if lists:  # the shard is on the device; drop the full row arrays
        arr = None
        torch.cuda.empty_cache()
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
    step_ms = [s_.elapsed_time(e_) for s_, e_ in zip(starts, ends)]
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
    _native.profile_enable(True)
    _native.profile_read()
    prof_steps = max(1, min(3, args.steps))
    for _ in range(prof_steps):
        l2_flush(flush)
        step()
    torch.cuda.synchronize()
    stages = _native.profile_read()
    _native.profile_enable(False)

    # ---- end to end through the public API with host buffers (pinned)
    from paper_1802_02422_b200.query import search_batch

    h2d = queries.nbytes
    d2h = nq * k * 8 + nq * 32
    qh = torch.from_numpy(queries).pin_memory()
    if not lists:  # every rank: its own batch through the public API
        qn = qh.numpy()
        oi = torch.empty((nq, k), dtype=torch.int32).pin_memory().numpy()
        od = torch.empty((nq, k), dtype=torch.float32).pin_memory().numpy()
        os_ = torch.empty((nq, 4), dtype=torch.int64).pin_memory().numpy()

        def e2e_step():
            search_batch(sx.dev, qn, params, k=k, out=(oi, od, os_))
            return oi
    else:  # H2D of the queries, sharded search + NCCL merge, D2H of the results
        oi_t = torch.empty((nq, k), dtype=torch.int32).pin_memory()
        od_t = torch.empty((nq, k), dtype=torch.float32).pin_memory()
        os_t = torch.empty((nq, 4), dtype=torch.int64).pin_memory()

        def e2e_step():
            qd = qh.to("cuda", non_blocking=True)
            i_, d_, s_ = sx.search_topk(qd, params, k)
            oi_t.copy_(i_, non_blocking=True)
            od_t.copy_(d_, non_blocking=True)
            os_t.copy_(s_, non_blocking=True)
            torch.cuda.synchronize()
            return oi_t.numpy()
    e2e_step()
    e2e_t = 0.0
    for _ in range(args.steps):
        l2_flush(flush)
        torch.cuda.synchronize()
        if world > 1:
            torch.distributed.barrier()
        t0 = time.perf_counter()
        got = e2e_step()
        e2e_t += time.perf_counter() - t0
    if world > 1:  # slowest rank
        t = torch.tensor([e2e_t], device="cuda")
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        e2e_t = float(t.item())
    e2e_qps = units * args.steps / e2e_t
    assert np.array_equal(got, ids_h), "e2e results differ from the device-resident run"

    sweep_on = (args.latency_sweep or w.get("latency_sweep", False)) and not args.no_sweeps
    sweep = latency_sweep(sx.dev, queries, w, k) if (sweep_on and world == 1) else None
    psweep = None
    sweep_spec = args.sweep if args.sweep is not None else ("" if args.no_sweeps else w.get("sweep", ""))
    if sweep_spec and world == 1:
        settings = [(int(a), float(b)) for a, b in (x.split(":") for x in sweep_spec.split(","))]
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
            # ncu DRAM bytes of one captured scan launch of this workload,
            # per query, scaled to this step's queries
            traffic = tr["dram_bytes_per_launch"] / tr["queries_per_launch"] * nq / shards
        except Exception:  # noqa: BLE001
            traffic = None
    gemm_ms, gemm_n = stages["probe_gemm"]
    probe_flops = 2.0 * w["k"] * w["d"] * nq
    step_stage_ms = {s_: v[0] / prof_steps for s_, v in stages.items() if v[1]}
    cfg = config_of(args, w, units)
    cfg.update({
        "queries_per_rank_step": nq,
        "recall@1": recall[1], "recall@10": recall[10], "recall@100": recall[100],
        "codes_scanned_mean": float(stats_h[:, 3].mean()),
        "l2": "flushed between steps (512 MB write); codes also exceed L2",
        "parallelism": (f"list-shard x{world} (NCCL all-gather + K7 merge)" if lists
                        else f"query-parallel x{world} (index replica per GPU, no collective)"
                        if world > 1 else "single GPU"),
        "build_s": build_s,
    })
    line = {
        "metric": "queries/sec at fixed recall@10 (synthetic, B200)",
        "value": qps,
        "unit": "queries/s",
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": total_ms / args.steps,
        "higher_is_better": True,
        "scaling": "strong" if lists else "weak",
        "vs_baseline": None,
        "dtype": "f32/f64 (u8 codes)",
        "data": ("synthetic: seeded SIFT-like uint8 gamma mixture, built on GPU"
                 if w.get("kind") == "sift_u8"
                 else f"synthetic: seeded gaussian mixture, noise={args.noise}, built on GPU"),
        "config": cfg,
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
        "roofline_probe": probe_roofline(w, nq, gemm_ms / prof_steps if gemm_n else None, peaks),
        "roofline_plan": plan_roofline(w, nq, step_stage_ms.get("plan_scores"), hbm_peak),
        "stage_ms_per_step": step_stage_ms,
        "gpu_launches": int(launches),
        "fallback_queries_per_step": fallbacks,
        **({"latency_sweep": sweep} if sweep else {}),
        **({"param_sweep": psweep} if psweep else {}),
        "plan_fallback_reasons_per_step": plan_reasons,
        "e2e": {"value": e2e_qps, "unit": "queries/s", "h2d_bytes_per_step": int(h2d),
                "d2h_bytes_per_step": int(d2h)},
        "clocks": clocks.summary(),
    }
    ref_recall = reference_recall(args.workload, args.noise)
    if ref_recall:
        line["reference_recall"] = ref_recall
    if world == 1 and not args.no_cpu_baseline:
        cpu = CpuOracle(arr, queries, w)
        cps, done, wall = cpu.rate(args.cpu_seconds)
        cpu.close()
        line["cpu_baseline"] = {"value": cps, "unit": "queries/s", "cores": cpu.cores, "kind": "port",
                                "sample": f"{done} of the {nq} step queries in {wall:.1f}s "
                                          f"(oracle port of search.py, exact probe, fork x{cpu.cores})"}
    return line


def plan_roofline(w, nq, ms, hbm_peak):
    """K3a (approximate group scores, the pruning's input) against HBM.  With
    the fused probe (K >= 2^17) it reads the fp16 rows of the P L neighbour
    centroids of the probed regions, 32 ceil(d / 32) x 2 bytes each, from the
    per-region packed copy; below that it gathers P L 2-byte scores from the
    score matrix (sector-bound, no byte roofline stated)."""
    if not ms or w["k"] < (1 << 17):
        return None
    row = -(-w["d"] // 32) * 32 * 2
    nbytes = float(nq) * w["nprobe"] * w["l"] * row
    gbs = nbytes / (ms / 1e3) / 1e9
    return {"kernel": "k_plan_scores_direct (K3a: fp16 neighbour rows, packed per region)",
            "bound": "hbm", "achieved": gbs, "peak": hbm_peak, "unit": "GB/s", "frac": gbs / hbm_peak,
            "algorithmic_bytes_per_step": nbytes, "kernel_ms_per_step": ms,
            "note": "peak = measured copy bandwidth (read + write); a read-only stream can exceed it"}


def probe_roofline(w, nq, gemm_ms, peaks):
    """The probe GEMM stage against its bounds.  K >= 2^17 runs the fused
    probe (probe_fused.cu: one fp16 tcgen05 product per term, 2 K d flops per
    query; the epilogue reads every fp32 accumulator from TMEM once, K x 4
    bytes per query; the MMA runs ceil((d + 2) / 16) k-steps of 16 columns:
    q.c plus the folded |c|^2 term, zero padded);
    smaller K the bf16x3 GEMM with fp16 score stores (probe_tc.cu)."""
    if not gemm_ms:
        return None
    flops = 2.0 * w["k"] * w["d"] * nq
    fused = w["k"] >= (1 << 17)
    peak = float(peaks.get("bf16_tflops", 1590.0))
    out = {"kernel": ("k_probe_filter (fused fp16 tcgen05 GEMM, threshold epilogue, no score store)"
                      if fused else "k_probe_gemm_tc (bf16x3 tcgen05 GEMM, fp16 score store)"),
           "unit": "TFLOP/s", "kernel_ms_per_step": gemm_ms,
           "achieved_tflops": flops / (gemm_ms / 1e3) / 1e12,
           "mma_tflops": (flops * (-(-(w["d"] + 2) // 16) * 16) / w["d"] if fused
                          else flops * 10.0 / 3.0) / (gemm_ms / 1e3) / 1e12,
           "peak_tflops_dense_bf16": peak}
    out["frac_algorithmic"] = out["achieved_tflops"] / peak
    out["frac_of_tensor_peak"] = out["mma_tflops"] / peak
    if fused:
        out["tmem_read_GBps"] = 4.0 * w["k"] * nq / (gemm_ms / 1e3) / 1e9
    return out


def reference_recall(workload, noise):
    """The reference's own recall@10 on the same data family, measured with
    the reference package (tools/reference_recall.py, committed result)."""
    path = os.path.join(ROOT, "profiles", "reference_recall.json")
    if not os.path.exists(path):
        return None
    try:
        return json.load(open(path))
    except Exception:  # noqa: BLE001
        return None


def run_reference(args, w):
    """The reference's CPU query path (oracle port of search.py:93-163 with
    the exact probe) on the host cores, same workload; each step is a
    bounded sample of 8 queries per core (rank 0 only)."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return None
    import torch

    torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", "0")))
    arr, queries, gt, _ = load_or_build(w, args.noise, args.seed, "cuda")
    torch.cuda.empty_cache()
    cpu = CpuOracle(arr, queries, w)
    del arr
    per = 8 * cpu.cores
    for _ in range(args.warmup):
        cpu.run(per)
    walls, done = [], 0
    for _ in range(args.steps):
        d, t = cpu.run(per)
        walls.append(t)
        done += d
    cpu.close()
    total = float(np.sum(walls))
    v = done / total
    return {
        "impl": "reference",
        "metric": "queries/sec at fixed recall@10 (synthetic, B200)",
        "value": v, "unit": "queries/s", "n_gpus": int(os.environ.get("WORLD_SIZE", "1")),
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * total / args.steps,
        "higher_is_better": True,
        "scaling": "strong" if args.layout == "lists" and int(os.environ.get("WORLD_SIZE", "1")) > 1 else "weak",
        "vs_baseline": None,
        "dtype": "f32/f64 (u8 codes)", "data": f"synthetic, noise={args.noise}",
        "config": dict(config_of(args, w, w["nq"]), queries_per_step_timed=per,
                       sample=f"each step: {per} of the {w['nq']} queries (8 per core)"),
        "cpu_baseline": {"value": v, "unit": "queries/s", "cores": cpu.cores, "kind": "port",
                         "sample": f"{done} queries over {args.steps} steps of {per}"},
        "e2e": {"value": v, "unit": "queries/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="c3", choices=sorted(WORKLOADS))
    ap.add_argument("--latency-sweep", action="store_true",
                    help="add BASELINE configs[4]'s batch x budget latency sweep (N=1; on by "
                         "default for c3)")
    ap.add_argument("--sweep", default=None,
                    help="nprobe:tau settings on the same index, e.g. 32:0.5,128:0.25 (N=1; "
                         "default: the workload's BASELINE sweep)")
    ap.add_argument("--no-sweeps", action="store_true", help="skip both sweeps")
    ap.add_argument("--noise", default="total", choices=["per_coord", "total"])
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--nprobe", type=int)
    ap.add_argument("--tau", type=float)
    ap.add_argument("--candidates", type=int)
    ap.add_argument("--cpu-seconds", type=float, default=20.0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--layout", default="lists", choices=["queries", "lists"],
                    help="N>1: list shards merged over NCCL (strong scaling, default) or "
                         "query-parallel replicas (weak scaling)")
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
