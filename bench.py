#!/usr/bin/env python3
"""bench.py -- exact-match queries/s on B200 (arXiv 1303.3692's hot path), one JSON line.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config C4] [--impl reference]
  torchrun --nproc-per-node N bench.py --gpus N ...          (one rank per GPU, NCCL)

A step is one pass of the hot path -- ``sa_match_order`` + ``sa_match_batch`` over this rank's whole
batch of packed reads (read ordering, bracket lookup, joint lo/hi binary search, interval write) --
with the index and the reads already resident in HBM.  The index build is off the timed path
(SURVEY.md Sec. 8(a) a1-a3).
Multi-GPU: the index is replicated and the job's Q reads are cut into N
contiguous slices, one per rank (strong scaling: C4 is "100M reads sharded over 1/2/4/8 GPUs";
``--weak`` gives every rank its own Q reads instead); no data-path collective; elapsed time is the
max over ranks (all_reduce MAX).  ``--gpus N`` without torchrun (WORLD_SIZE unset) starts the N
ranks itself.

`--impl reference` times the CPU oracle (oracle/: the streaming counting oracle, no suffix array)
on a bounded sample of the same workload on this box's host cores.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import socket
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import synth  # noqa: E402

METRIC = "exact-match queries/sec and achieved HBM GB/s at 1/2/4/8 B200"
UNIT = "queries/s"
BUCKET_MAX_Q = 16_000_000  # order_method auto: bucket placement up to this many reads per GPU


def log(*a):
    if int(os.environ.get("RANK", "0")) == 0:
        print("[bench]", *a, file=sys.stderr, flush=True)


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=30)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--config", default="C4", choices=sorted(synth.CONFIGS))
    ap.add_argument("--m", type=int, default=None, help="C5 read length (16..1000)")
    ap.add_argument("--q", type=int, default=None, help="override the job's reads Q (split over the ranks)")
    ap.add_argument("--weak", action="store_true",
                    help="weak scaling: every rank matches its own Q reads (default: the Q reads are split over the ranks)")
    ap.add_argument("--k", type=int, default=0, help="k-mer bracket k (0 = auto: floor(log4 n)+1, <= 16)")
    ap.add_argument("--layout", default="rec32", choices=["rec16", "rec32", "plain"],
                    help="SA layout: 16-byte records caching 48 bases (default), 32-byte records caching 112 "
                         "bases, or a plain uint32 SA")
    ap.add_argument("--subtables", action="store_true",
                    help="second-level (k+4)-base tables for k-mer buckets of > 32 suffixes (SA_INDEX_SUBTABLE)")
    ap.add_argument("--build", default="doubling", choices=["doubling", "dc3"],
                    help="suffix-array construction (untimed): prefix doubling or the paper's DC3")
    ap.add_argument("--no-order", action="store_true", help="skip the read-ordering step (a5)")
    ap.add_argument("--chunks", type=int, default=1,
                    help="split the batch into this many chunks, ordering chunk i+1 on a second stream while "
                         "chunk i is searched")
    ap.add_argument("--partition", action="store_true",
                    help="SURVEY.md 8(f) f4: each rank holds 1/WORLD_SIZE of the index (route-key range) and reads "
                         "are exchanged with all-to-alls (shard.partitioned_match)")
    ap.add_argument("--tree", action="store_true",
                    help="time the flattened suffix tree walk (sa_tree_match, SURVEY.md 8(f) f3) instead of the SA search")
    ap.add_argument("--order-bases", type=int, default=12, help="bases of the read-ordering key (1..16)")
    ap.add_argument("--defer", type=int, default=0,
                    help="SA_MATCH_DEFER: reads whose k-mer bracket holds more than 2^DEFER suffixes are searched "
                         "in a second, full-warp pass (0 = off)")
    ap.add_argument("--order-method", choices=["auto", "sort", "buckets"], default="sort",
                    help="read ordering: the stable radix sort, bucket placement (SA_ORDER_BUCKETS), or auto "
                         "(buckets when the rank's batch is <= BUCKET_MAX_Q reads)")
    ap.add_argument("--rows-ordered", action="store_true",
                    help="the ordering step also gathers the read rows into order (SA_MATCH_ROWS_ORDERED)")
    ap.add_argument("--cooperative", action="store_true",
                    help="SA_MATCH_COOPERATIVE: reads over 128 bases searched by 8/16/32-lane groups")
    ap.add_argument("--bucket-tree", action="store_true",
                    help="SA_INDEX_BUCKET_TREE: line-packed binary-search trees for k-mer buckets of >= 32 suffixes")
    ap.add_argument("--smem-tree", type=int, default=0,
                    help="SA_MATCH_SMEM_TREE: levels (1..12) of the per-CTA shared-memory top tree staged by TMA "
                         "(SURVEY.md 8(a) a3(ii)); 0 = off")
    ap.add_argument("--no-graph", dest="graph", action="store_false",
                    help="launch the step's kernels one by one instead of replaying them from two CUDA graphs")
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--e2e-chunk", type=int, default=0, help="reads per chunk of the host pipeline (0 = library default)")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-locate", action="store_true")
    ap.add_argument("--dist-backend", default="nccl", choices=["nccl", "gloo"],
                    help="process-group backend (gloo only to test the multi-rank path with ranks sharing a GPU)")
    ap.add_argument("--cpu-seconds", type=float, default=15.0,
                    help="target CPU time of the cpu_baseline's single-thread sample (and of the reference arm's step)")
    ap.add_argument("--cpu-sample", type=int, default=1_000_000, help="cpu_baseline: at most this many reads")
    return ap.parse_args()


def workload(args):
    cfg = synth.CONFIGS[args.config]
    if args.config == "C5":
        cfg = cfg.with_m(args.m or 100)
    if args.q:
        cfg = synth.Config(cfg.name, cfg.ref_kind, cfg.n, cfg.ref_seed, args.q, cfg.m_min, cfg.m_max, cfg.p_random,
                           cfg.p_mut_read, cfg.read_seed, cfg.description)
    return cfg


def config_json(cfg, world, reads_per_gpu, weak=False, k=None, index_bytes=None):
    d = {"workload": f"{cfg.name}: {cfg.description}", "n_bases": cfg.n, "reads_per_gpu": reads_per_gpu,
         "global_reads": reads_per_gpu * world if weak else cfg.Q,
         "read_len": (cfg.m_min if cfg.m_min == cfg.m_max else [cfg.m_min, cfg.m_max]),
         "parallelism": f"replicated index x{world}, " + (f"{cfg.Q} reads per rank (weak)" if weak else
                                                           f"{cfg.Q} reads split in {world} contiguous shards") +
                        " (no data-path collective)"}
    if index_bytes is not None:
        # what one step reads at random vs the 126 MB L2 (inputs larger than L2 need no flush)
        resident = index_bytes + reads_per_gpu * cfg.stride * 8
        d["l2"] = (f"inputs larger than L2 (index {index_bytes / 1e9:.2f} GB + reads >> 126 MB); no flush"
                   if index_bytes > 126e6 else
                   f"index fits L2 ({index_bytes / 1e6:.1f} MB <= 126 MB: an L2-resident workload); no flush")
        d["resident_bytes"] = resident
    if k is not None:
        d["kmer_k"] = k
    return d


# ---------------------------------------------------------------------------------------------
class ClockSampler:
    """Samples SM clock + throttle reasons through NVML during the timed region."""
    REASONS = {0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap", 0x8: "hw_slowdown",
               0x10: "sync_boost", 0x20: "sw_thermal_slowdown", 0x40: "hw_thermal_slowdown",
               0x80: "hw_power_brake_slowdown", 0x100: "display_clock_setting"}

    def __init__(self, device_index):
        self.samples, self.reasons = [], 0
        self.max_mhz = None
        self._stop = threading.Event()
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(device_index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
        except Exception as e:  # pragma: no cover
            self.nv = None
            log("NVML unavailable:", e)

    def _run(self):
        while not self._stop.is_set():
            try:
                self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
                self.reasons |= self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
            except Exception:
                pass
            time.sleep(0.01)

    def __enter__(self):
        if self.nv:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *exc):
        if self.nv:
            self._stop.set()
            self.t.join()

    def result(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": ["unavailable"]}
        rs = [name for bit, name in self.REASONS.items() if self.reasons & bit and name != "gpu_idle"]
        return {"sm_mhz": statistics.median(self.samples), "sm_max_mhz": self.max_mhz, "reasons": rs,
                "samples": len(self.samples)}


def measured_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


def survey_bytes_per_query(n, m):
    """SURVEY.md 8(d)'s algorithmic ("useful") bytes per query, the per-unit figure the roofline's `achieved`
    is defined on: D_eff x (4 B SA entry + ceil((l+1)/4) = 1 B of text at l ~ 1/2 base decided per level)
    + ceil(m/4) B verify + ceil(m/4) B query + 8 B result, D_eff = ceil(log2(n+1)) (the textbook search's
    full-range depth).  C4, m = 100: 32 x 5 + 25 + 25 + 8 = 218 B."""
    d_eff = math.ceil(math.log2(n + 1))
    return d_eff * 5.0 + 2.0 * math.ceil(m / 4.0) + 8.0


def sector_bytes_per_query(m, probes, text_windows):
    """The 32-B-sector access model of r01 (kept for continuity): bracket pair + one sector per probe and
    per text window + the read row + the 8-B result."""
    return 32.0 + 32.0 * probes + 32.0 * text_windows + max(32.0, math.ceil(m / 4.0)) + 8.0


def traffic_entry(key):
    """DRAM bytes per read (read + write) of k_match from the committed ncu --set full capture of this exact
    configuration (profiles/traffic.json, written from the profile of the same commit), or None."""
    try:
        with open(os.path.join(ROOT, "profiles", "traffic.json")) as f:
            t = json.load(f)
        e = t.get(key)
        return e if isinstance(e, dict) else None
    except Exception:
        return None


def cpu_model():
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return "unknown"


def free_port():
    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        return so.getsockname()[1]


def self_launch(args):
    """`--gpus N` without torchrun: start N ranks of this script (RANK / WORLD_SIZE / LOCAL_RANK /
    MASTER_* set as torchrun would, rendezvous on 127.0.0.1).  Rank 0 prints the JSON line.  If a rank
    fails, the others are stopped (by their own process handles) and its exit code is returned."""
    port = free_port()
    procs = []
    for r in range(args.gpus):
        env = dict(os.environ, RANK=str(r), WORLD_SIZE=str(args.gpus), LOCAL_RANK=str(r),
                   LOCAL_WORLD_SIZE=str(args.gpus), MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        procs.append(subprocess.Popen([sys.executable, os.path.abspath(__file__)] + sys.argv[1:], env=env))
    rc = 0
    live = list(procs)
    while live:
        for p in list(live):
            code = p.poll()
            if code is None:
                continue
            live.remove(p)
            if code != 0 and rc == 0:
                rc = code
                for q in live:
                    q.terminate()
        time.sleep(0.2)
    return rc


# ---------------------------------------------------------------------------------------------
def run_reference_arm(args):
    """The CPU oracle on this box's host cores (rank 0 only; it never loads libsa)."""
    import oracle
    from paper_1303_3692_b200 import shard
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    cfg = workload(args)
    world = int(os.environ.get("WORLD_SIZE", str(args.gpus)))
    t0 = time.time()
    ref = cfg.reference()
    S = oracle.encode(ref)
    log(f"reference generated+encoded in {time.time() - t0:.1f}s")
    cores = oracle.max_threads()
    # keep the whole --steps/--warmup run within a few minutes
    s = sample_size(cfg, cores, min(args.cpu_seconds, 150.0 / max(1, args.steps + args.warmup)))
    times = []
    for it in range(args.warmup + args.steps):
        # each step: a fresh bounded sample of the same read stream
        words, lens = cfg.reads(ref, q_begin=it * s, q_count=s)
        t = time.perf_counter()
        oracle.count_batch(S, words, lens)
        dt = time.perf_counter() - t
        if it >= args.warmup:
            times.append(dt)
    tot = sum(times)
    v = s * len(times) / tot
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": 1e3 * tot / len(times), "higher_is_better": True,
            "scaling": "weak" if args.weak else "strong", "vs_baseline": None, "dtype": "u8", "data": "synthetic",
            "config": config_json(cfg, world, shard.shard(0, world, cfg.Q, weak=args.weak)[1], weak=args.weak),
            "cpu_baseline": {"value": v, "unit": UNIT, "cores": cores, "kind": "oracle",
                             "sample": f"{s} reads per step of the {cfg.name} read stream, streaming counting "
                                       f"oracle over all {cfg.n} suffixes (no suffix array)"},
            "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def sample_size(cfg, cores, seconds):
    """Reads per oracle sample so that one streaming pass costs ~`seconds` on `cores` threads.
    Cost model: n * log2(2s) suffix-vs-key compares at ~6 ns each (measured on the dev box)."""
    per_pass = cfg.n * 6e-9 / max(1, cores)
    if per_pass <= 0:
        return 64
    lg = max(1.0, seconds / per_pass)
    s = int(min(2 ** min(lg, 20) / 2, 1 << 16))
    return max(16, min(s, cfg.Q))


def cpu_baseline(cfg, ref, idx, words, lens, got, seconds, max_sample):
    """SURVEY.md §8(d) / BASELINE.md "CPU-baseline plan": the oracle's textbook lower/upper-bound search
    (oracle_search_batch, P:L173-230 corrected) over the GPU-built suffix array, passed as data, on a
    sample of this run's reads, single-threaded and on all host cores; rates extrapolated to the batch.
    The sample's intervals are also compared with the GPU's (`agrees_with_gpu`)."""
    import oracle
    S = oracle.encode(ref)
    t0 = time.perf_counter()
    sa_host = idx.export_sa()
    export_s = time.perf_counter() - t0
    cores = oracle.max_threads()
    Q = words.shape[0]
    lw = None if lens is None else lens
    # calibrate the single-thread rate on a small prefix, then size the sample to ~`seconds`
    c = min(Q, 2000)
    t = time.perf_counter()
    oracle.search_batch(S, sa_host, words[:c], None if lw is None else lw[:c], fixed_len=cfg.m_max, nthreads=1)
    per = max(1e-9, (time.perf_counter() - t) / c)
    s1 = int(max(c, min(max_sample, Q, seconds / per)))
    t = time.perf_counter()
    r1 = oracle.search_batch(S, sa_host, words[:s1], None if lw is None else lw[:s1], fixed_len=cfg.m_max, nthreads=1)
    d1 = time.perf_counter() - t
    sa_ = min(max_sample, Q)
    t = time.perf_counter()
    ra = oracle.search_batch(S, sa_host, words[:sa_], None if lw is None else lw[:sa_], fixed_len=cfg.m_max,
                             nthreads=cores)  # (explicit: the 1-thread call left OpenMP at 1 thread)
    da = time.perf_counter() - t
    agree = bool(np.array_equal(ra.astype(np.uint32), got[:sa_]) and np.array_equal(r1.astype(np.uint32), got[:s1]))
    v1, va = s1 / d1, sa_ / da
    return {"value": va, "unit": UNIT, "cores": cores, "kind": "oracle", "cpu_model": cpu_model(),
            "sample": f"first {sa_} reads of this run's {cfg.name} batch (all cores) / first {s1} (1 thread): "
                      f"textbook lower/upper-bound binary search (oracle_search_batch) over the GPU-built suffix "
                      f"array passed as data ({cfg.n} suffixes); rates extrapolated to the batch",
            "extrapolated": True,
            "single_thread": {"value": v1, "sample_reads": s1, "seconds": d1},
            "all_cores": {"value": va, "sample_reads": sa_, "seconds": da, "threads": cores},
            "projected_seconds_full_batch": {"1_thread": Q / v1, "all_cores": Q / va},
            "sa_export_seconds": export_s, "agrees_with_gpu": agree}


# ---------------------------------------------------------------------------------------------
def main():
    args = parse()
    if args.impl == "reference":
        run_reference_arm(args)
        return
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(self_launch(args))
    import torch
    import torch.distributed as dist
    import paper_1303_3692_b200 as sa
    from paper_1303_3692_b200 import shard

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        raise SystemExit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}: launch with torchrun "
                         f"--nproc-per-node {args.gpus}, or without torchrun to let bench.py start the ranks")
    ndev = torch.cuda.device_count()
    if local >= ndev:  # test mode only (--dist-backend gloo): several ranks share the visible GPUs
        if args.dist_backend == "nccl":
            raise RuntimeError(f"LOCAL_RANK {local} but only {ndev} GPUs visible")
        local = local % ndev
    torch.cuda.set_device(local)
    numa = shard.bind_numa_local(local)  # before any pinned host buffer is allocated and touched
    if world > 1:
        if args.dist_backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group("gloo")
    dev = torch.device("cuda", local)
    cfg = workload(args)

    # ---- inputs + index (untimed) ----
    t0 = time.time()
    ref = cfg.reference()
    log(f"{cfg.name}: reference of {cfg.n} bases generated in {time.time() - t0:.1f}s")
    t0 = time.time()
    k_auto = args.k
    if not k_auto:  # the library's auto k: floor(log4 n) + 1, at most 16
        k_auto = 1
        while k_auto < 16 and 4 ** k_auto <= cfg.n:
            k_auto += 1
    part = (rank, world, min(12, k_auto - 1)) if args.partition else None  # route key: < k, <= 12 bases
    idx = sa.Index(ref, k=args.k, device=local, layout=args.layout, build=args.build, part=part,
                   subtables=args.subtables, bucket_tree=args.bucket_tree)
    torch.cuda.synchronize()
    build_s = time.time() - t0
    log(f"index built in {build_s:.1f}s: k={idx.k}, {idx.device_bytes / 1e9:.2f} GB resident")
    tree = None
    if args.tree:
        t1 = time.time()
        tree = sa.Tree(idx)
        log(f"flattened suffix tree: {tree.nodes} nodes, {tree.device_bytes / 1e9:.2f} GB, {time.time() - t1:.1f}s")
    t0 = time.time()
    q_begin, Q = shard.shard(rank, world, cfg.Q, weak=args.weak)  # this rank's contiguous slice of the reads
    stride = cfg.stride
    fixed = cfg.m_max if cfg.m_min == cfg.m_max else None
    words_h = torch.empty((Q, stride), dtype=torch.int64, pin_memory=True)
    lens_h = torch.empty(Q, dtype=torch.int32, pin_memory=True)
    cfg.reads(ref, q_begin=q_begin, q_count=Q, words_out=words_h.numpy().view(np.uint64),
              lens_out=lens_h.numpy().view(np.uint32))
    words = words_h.to(dev, non_blocking=True)
    lens = None if fixed else lens_h.to(dev, non_blocking=True)
    out = torch.empty((Q, 2), dtype=torch.int32, device=dev)
    torch.cuda.synchronize()
    log(f"{Q} reads/rank generated + uploaded in {time.time() - t0:.1f}s")

    stream = torch.cuda.current_stream()
    presort = not args.no_order
    # the read ordering (a5): the stable radix sort, or bucket placement (SA_ORDER_BUCKETS) for batches
    # whose permutation + 4^12 counters stay in L2 ("auto": Q <= BUCKET_MAX_Q reads per GPU)
    buckets = presort and (args.order_method == "buckets" or
                           (args.order_method == "auto" and Q <= BUCKET_MAX_Q and args.order_bases <= 12))
    ws = torch.empty(max(1, idx.workspace_size(Q, stride, sa.SA_MATCH_STATS | sa.SA_MATCH_PRESORT),
                         idx.workspace_size(Q, stride, sa.SA_MATCH_PRESORT | sa.SA_MATCH_DEFER),
                         idx.order_workspace_size(Q, args.order_bases, buckets=buckets)),
                     dtype=torch.uint8, device=dev)
    perm = torch.empty(Q, dtype=torch.int32, device=dev) if presort else None
    rows_ordered = presort and args.rows_ordered
    owords = torch.empty_like(words) if rows_ordered else None
    olens = torch.empty_like(lens) if (rows_ordered and lens is not None) else None
    ev = [tuple(torch.cuda.Event(enable_timing=True) for _ in range(2)) for _ in range(args.steps)]

    chunks = max(1, args.chunks) if presort and not rows_ordered and tree is None else 1
    streams = [stream] + [torch.cuda.Stream(device=dev) for _ in range(1 if chunks > 1 else 0)]
    bounds = [Q * c // chunks for c in range(chunks + 1)]
    ws_c = [ws] + [torch.empty_like(ws) for _ in range(1 if chunks > 1 else 0)]

    def step(i=None):
        # one pass of the hot path: [read ordering (a5)] -> bracket + joint lo/hi search + write (a6-a9)
        if args.partition:
            if i is not None:
                ev[i][0].record(stream)
            shard.partitioned_match(idx, words, lens, fixed_len=fixed, out=out)
            if i is not None:
                ev[i][1].record(stream)
            return
        if chunks > 1:
            # order chunk c on stream c%2 while chunk c-1 is searched on the other; results join at the end
            if i is not None:
                ev[i][0].record(stream)
            streams[1].wait_stream(stream)
            for c in range(chunks):
                sc, q0, q1 = streams[c % 2], bounds[c], bounds[c + 1]
                lw = None if lens is None else lens[q0:q1]
                idx.order(words[q0:q1], lw, fixed_len=fixed, out=perm[q0:q1], stream=sc, workspace=ws_c[c % 2],
                          key_bases=args.order_bases)
                idx.match(words[q0:q1], lw, fixed_len=fixed, out=out[q0:q1], stream=sc, workspace=ws_c[c % 2],
                          order=perm[q0:q1])
            stream.wait_stream(streams[1])
            if i is not None:
                ev[i][1].record(stream)  # chunked: the "launch" time is the whole overlapped step
            return
        if presort:
            idx.order(words, lens, fixed_len=fixed, out=perm, stream=stream, workspace=ws, key_bases=args.order_bases,
                      ordered_words=owords, ordered_lens=olens, buckets=buckets)
        if i is not None:
            ev[i][0].record(stream)
        if tree is not None:
            tree.match(words, lens, fixed_len=fixed, out=out, stream=stream, order=perm)
        elif rows_ordered:
            idx.match(owords, olens, fixed_len=fixed, out=out, stream=stream, workspace=ws, order=perm, rows_ordered=True,
                      cooperative=args.cooperative)
        else:
            idx.match(words, lens, fixed_len=fixed, out=out, stream=stream, workspace=ws, order=perm,
                      cooperative=args.cooperative, smem_tree=args.smem_tree, tree_key_bases=args.order_bases,
                      defer=args.defer)
        if i is not None:
            ev[i][1].record(stream)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()

    graphs = None
    if args.graph and presort and chunks == 1 and not (args.partition or tree is not None or rows_ordered or
                                                       args.smem_tree or args.cooperative):
        # the step's launches (key extraction, CUB's sort kernels, k_match) captured once and replayed:
        # no per-launch CPU work or inter-kernel launch gaps inside a step
        g_order, g_match = torch.cuda.CUDAGraph(), torch.cuda.CUDAGraph()
        cs = torch.cuda.Stream(device=dev)
        cs.wait_stream(stream)
        with torch.cuda.graph(g_order, stream=cs):
            idx.order(words, lens, fixed_len=fixed, out=perm, stream=cs, workspace=ws, key_bases=args.order_bases,
                      buckets=buckets)
        with torch.cuda.graph(g_match, stream=cs):
            idx.match(words, lens, fixed_len=fixed, out=out, stream=cs, workspace=ws, order=perm,
                      smem_tree=args.smem_tree, tree_key_bases=args.order_bases, defer=args.defer)
        stream.wait_stream(cs)
        graphs = (g_order, g_match)

        def step(i=None):  # noqa: F811  (the same step, replayed from the graphs)
            g_order.replay()
            if i is not None:
                ev[i][0].record(stream)
            g_match.replay()
            if i is not None:
                ev[i][1].record(stream)

        for _ in range(args.warmup):
            step()
        torch.cuda.synchronize()

    # ---- timed region ----
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    sampler = ClockSampler(local)
    with sampler:
        t_start = torch.cuda.Event(enable_timing=True)
        t_end = torch.cuda.Event(enable_timing=True)
        t_start.record(stream)
        for i in range(args.steps):
            step(i)
        t_end.record(stream)
        torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    elapsed_ms = t_start.elapsed_time(t_end)
    launch_ms = [a.elapsed_time(b) for a, b in ev]
    elapsed_ms = shard.max_over_ranks(elapsed_ms, dev)
    # per-shard summary gathered over NCCL (the only collective): hits, sum of counts, checksum
    summary_all = shard.gather_summaries(shard.summarize(out))

    global_reads = shard.all_reduce_sum(Q, dev)  # the reads all ranks matched per step
    total_reads = global_reads * args.steps
    value = total_reads / (elapsed_ms * 1e-3)
    ms_per_step = elapsed_ms / args.steps

    m_alg = cfg.m_max if fixed else (cfg.m_min + cfg.m_max) / 2
    avg_launch_s = statistics.mean(launch_ms) * 1e-3
    peak, peak_src = measured_peaks()
    traffic_key = f"{cfg.name}/{args.layout}/k{idx.k}/Q{Q}" + ("/tree" if args.tree else "")
    traffic_e = traffic_entry(traffic_key)

    line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True,
            "scaling": "weak" if args.weak else "strong", "vs_baseline": None, "dtype": "u64", "data": "synthetic",
            "config": config_json(cfg, world, Q, weak=args.weak, k=idx.k, index_bytes=idx.device_bytes),
            "numa": numa,
            "clocks": sampler.result(),
            "gpu_launches": args.steps * ((3 if buckets else 2) if presort else 1) + (args.steps if args.defer else 0),
            "defer_log2": args.defer,
            "library_launches_per_step": ("CUB exclusive scan of the 4^key_bases bucket counters" if buckets else
                                          f"CUB onesweep radix sort ({(2 * args.order_bases + 7) // 8} passes)"
                                          if presort else 0),
            "order_method": ("buckets (SA_ORDER_BUCKETS)" if buckets else "stable radix sort") if presort else None,
            "launch_ms": {"min": min(launch_ms), "median": statistics.median(launch_ms), "max": max(launch_ms)},
            "shards": summary_all, "layout": args.layout, "smem_tree_levels": args.smem_tree,
            "bucket_tree": args.bucket_tree, "cuda_graphs": graphs is not None, "read_order": f"sorted by first {args.order_bases} bases (sa_match_order, timed)" if presort else "as given",
            "index_bytes": idx.device_bytes,
            "index_build": {"seconds": build_s, "sa_algorithm": args.build,
                            "note": "untimed: upload + pack + suffix array + k-mer table + records"}}

    if not args.partition:
        # ---- search statistics (untimed instrumented launch): steps and text windows per read ----
        chk = torch.empty_like(out)
        if tree is not None:  # the walk must give the SA search's intervals
            ref_out = idx.match(words, lens, fixed_len=fixed, stream=stream)
            torch.cuda.synchronize()
            if not torch.equal(ref_out, out):
                raise RuntimeError("suffix-tree walk disagrees with the SA search")
            line["tree"] = {"nodes": tree.nodes, "bytes": tree.device_bytes, "kernel": "k_tree_match"}
            del ref_out
        if rows_ordered:
            _, st = idx.match(owords, olens, fixed_len=fixed, out=chk, stream=stream, want_stats=True, workspace=ws,
                              order=perm, rows_ordered=True)
        else:  # (with --chunks the permutation is chunk-local: any order gives the same intervals)
            _, st = idx.match(words, lens, fixed_len=fixed, out=chk, stream=stream, want_stats=True, workspace=ws,
                              order=perm if chunks == 1 else None)
        torch.cuda.synchronize()
        if not torch.equal(chk, out):
            raise RuntimeError("instrumented launch disagrees with the timed launches")
        stv = st[0].to(torch.int64) & 0xFFFFFFFF
        ubytes = (st[1].to(torch.int64) & 0xFFFFFFFF).double()
        steps_t, texts_t = (stv & 0xFFFF).double(), (stv >> 16).double()
        line["search_stats"] = {"mean_steps": float(steps_t.mean()), "mean_text_windows": float(texts_t.mean()),
                                "p99_steps": float(torch.quantile(steps_t[:1 << 20], 0.99)),
                                "max_steps": float(steps_t.max()),
                                "mean_algorithmic_bytes": float(ubytes.mean())}

        # ---- roofline of the dominant kernel (k_match; the ordering sort is CUB's) ----
        # achieved = SURVEY.md 8(d)'s per-query algorithmic bytes (survey_bytes_per_query: D_eff = 32 levels at
        # C4) x Q / the mean k_match launch time of the timed steps.  The bytes THIS method moves usefully (the
        # k-mer table resolves ~28 of the 32 levels; counted per read by the instrumented launch of this very
        # batch, SA_MATCH_STATS) are reported beside it as method_bytes_per_query / method_frac.
        bpq_m = line["search_stats"]["mean_algorithmic_bytes"]
        bpq = survey_bytes_per_query(cfg.n, m_alg)
        if tree is not None:
            line["search_stats"]["note"] = "counts of the SA search (the timed kernel is the tree walk)"
        achieved = bpq * Q / avg_launch_s / 1e9
        traffic = traffic_e["dram_bytes_per_read"] * Q if traffic_e else None
        roofline = {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                    "traffic": traffic, "kernel": "k_tree_match" if tree is not None else "k_match",
                    "algorithmic_bytes_per_query": bpq,
                    "algorithmic_bytes_formula": "SURVEY.md 8(d): D_eff x (4 B SA entry + 1 B text) + ceil(m/4) verify "
                                                 "+ ceil(m/4) query + 8 result, D_eff = ceil(log2(n+1))",
                    "method_bytes_per_query": bpq_m,
                    "method_frac": bpq_m * Q / avg_launch_s / 1e9 / peak,
                    "method_bytes_formula": "ceil(m/4) read + 8 table pair + sum over this method's probes of "
                                            "(4 B SA entry + ceil(decided bases/4)) + 8 result, decided bases = "
                                            "from min(lcp_L, lcp_R) to the first difference (all m at a match); "
                                            "per read from SA_MATCH_STATS on this batch",
                    "measured_counts": {"probes_per_query": line["search_stats"]["mean_steps"],
                                        "text_windows_per_query": line["search_stats"]["mean_text_windows"]},
                    "sector_bytes_per_query": sector_bytes_per_query(m_alg, line["search_stats"]["mean_steps"],
                                                                     line["search_stats"]["mean_text_windows"]),
                    "peak_source": peak_src, "launch_ms_mean": avg_launch_s * 1e3}
        if tree is not None:
            roofline["note"] = "bytes of the SA search; the tree walk moves one 32-B node + one text window per level"
        if traffic_e:
            roofline["traffic_source"] = traffic_e.get("source")
            roofline["traffic_bytes_per_query"] = traffic_e["dram_bytes_per_read"]
            roofline["traffic_GBps"] = traffic / avg_launch_s / 1e9
            roofline["traffic_frac"] = roofline["traffic_GBps"] / peak
        else:
            roofline["traffic_source"] = f"no committed ncu capture for {traffic_key} (profiles/traffic.json)"
        line["roofline"] = roofline
        del st, chk

    # ---- locate (separate call): positions SA[lo..hi) of the reads ----
    # Repeat-rich references give some reads 10^5+ occurrences, so the located prefix of the batch is
    # capped at 2^30 positions (4 GiB); the line says how many reads and positions were located.
    if args.partition:  # the batch was answered across ranks: no per-rank stats / locate / e2e
        args.no_locate = args.no_e2e = True
        line["partition"] = idx.part_info()
        line["partition"].pop("part_keys")
    if not args.no_locate:
        torch.cuda.synchronize()
        l0, l1, l2 = (torch.cuda.Event(enable_timing=True) for _ in range(3))
        l0.record(stream)
        offs = idx.locate_offsets(out, stream=stream)
        l1.record(stream)
        cap = 1 << 30
        n_loc = int(torch.searchsorted(offs, torch.tensor([cap], device=dev, dtype=torch.int64), right=True).item()) - 1
        n_loc = max(0, min(Q, n_loc))
        npos_alloc = int(offs[n_loc].item())
        pos = torch.empty(npos_alloc, dtype=torch.int32, device=dev)  # allocated outside the timed call
        torch.cuda.synchronize()
        l1b = torch.cuda.Event(enable_timing=True)
        l1b.record(stream)
        idx.locate_positions(out, offs, n_reads=n_loc, stream=stream, out=pos)
        l2.record(stream)
        torch.cuda.synchronize()
        npos = int(pos.numel())
        line["locate"] = {"offsets_ms": l0.elapsed_time(l1), "gather_ms": l1b.elapsed_time(l2),
                          "reads_located": n_loc, "positions": npos, "total_positions_all_reads": int(offs[Q].item()),
                          "gather_GBps": npos * 4 * 2 / max(1e-9, l1b.elapsed_time(l2) * 1e-3) / 1e9}
        del offs, pos

    # ---- random-gather microbenchmark (the random-access roofline's denominator; untimed) ----
    # R_rand = the best of the load forms the microbenchmark offers (plain, .nc, .nc.L1::no_allocate) for
    # independent random 32-B loads over 16 GiB, measured in this run.
    if rank == 0:
        try:
            modes = {"ld": 0, "ld.global.nc": 10, "ld.global.nc.L1::no_allocate": 13}
            rgs = {name: sa.random_gather(local, buffer_bytes=16 << 30, access_bytes=32, n_threads=148 * 2048 * 2,
                                          loads=64, dependent=mode) for name, mode in modes.items()}
            best = max(rgs, key=lambda k_: rgs[k_]["Gaccess_per_s"])
            rg = rgs[best]
            line["random_gather_32B"] = {"GBps": rg["GBps"], "Gsectors_per_s": rg["Gaccess_per_s"], "best_mode": best,
                                         "by_mode_Gaccess_per_s": {k_: v["Gaccess_per_s"] for k_, v in rgs.items()},
                                         "note": "independent random 32-B loads over 16 GiB, 606k threads x 64"}
            if "roofline" in line and "search_stats" in line:
                # q/s ceiling = R_rand / random accesses per read.  A read's accesses: the
                # read row (through the ordering), the bracket-table pair, one record per probe, one text
                # window per window, the result store.  Each random access moves a 128-B DRAM line on this
                # B200, so the line rate during k_match is compared with R_rand x 128 B.
                ss = line["search_stats"]
                apq = 3.0 + ss["mean_steps"] + ss["mean_text_windows"]
                ceiling = rg["Gaccess_per_s"] * 1e9 / apq
                kernel_qps = Q / avg_launch_s
                rr = {"R_rand_Gaccess_per_s": rg["Gaccess_per_s"], "accesses_per_query": apq,
                      "ceiling_queries_per_s": ceiling, "kernel_queries_per_s": kernel_qps,
                      "frac": kernel_qps / ceiling,
                      "note": "ceiling = every access an independent random access; frac > 1 is the line sharing "
                              "the read ordering buys (neighbouring reads touch the same table / record lines); "
                              "line_frac = DRAM line rate of k_match (ncu traffic) / (R_rand x 128 B); with the 64-B "
                              "row / table fetches of large batches a lower bound on its access rate"}
                if line["roofline"].get("traffic_GBps"):
                    rr["dram_line_GBps"] = line["roofline"]["traffic_GBps"]
                    rr["line_frac"] = line["roofline"]["traffic_GBps"] / (rg["Gaccess_per_s"] * 128.0)
                line["random_access_roofline"] = rr
        except Exception as e:
            line["random_gather_32B"] = {"error": str(e)}

    # ---- e2e: the same match through the C ABI with HOST buffers (copies inside the timed region) ----
    # Fixed-length reads travel in the dense layout (2 bits/base, 25 B per 100-bp read); the host
    # pipeline streams chunks H2D -> match -> D2H on two streams (sa_match_batch_host).
    if not args.no_e2e:
        dense = fixed is not None and Q % 32 == 0
        if dense:
            nwords = Q // 32 * cfg.m_max
            dw = torch.empty(nwords, dtype=torch.int64, pin_memory=True)
            cfg.reads(ref, q_begin=q_begin, q_count=Q, words_out=dw.numpy().view(np.uint64), dense=True)
            wn, ln, h2d = dw.numpy(), None, nwords * 8
        else:
            wn, ln = words_h.numpy(), (None if fixed else lens_h.numpy())
            h2d = Q * stride * 8 + (0 if fixed else Q * 4)
        out_h = torch.empty((Q, 2), dtype=torch.int32, pin_memory=True)
        on = out_h.numpy()
        kw = {"n_reads": Q} if dense else {}
        kw["chunk"] = args.e2e_chunk
        idx.match_host(wn, ln, fixed_len=fixed, out=on, **kw)  # warm-up (allocates staging)
        e2e_steps = max(1, min(args.steps, 5))
        if world > 1:
            dist.barrier()
        t = time.perf_counter()
        for _ in range(e2e_steps):
            idx.match_host(wn, ln, fixed_len=fixed, out=on, **kw)
        dt = time.perf_counter() - t
        dt = shard.max_over_ranks(dt, dev)
        if not np.array_equal(on.view(np.uint32), out.cpu().numpy().view(np.uint32)):
            raise RuntimeError("host-buffer path disagrees with the device path")
        line["e2e"] = {"value": global_reads * e2e_steps / dt, "unit": UNIT, "h2d_bytes_per_step": h2d,
                       "d2h_bytes_per_step": Q * 8, "steps": e2e_steps,
                       "layout": "dense 2-bit stream" if dense else f"{stride} words per read",
                       "path": "sa_match_batch_host (pinned host buffers, 2 streams, "
                               f"{args.e2e_chunk or 2 << 20}-read chunks, each ordered)",
                       "overlapped_ms_per_step": dt * 1e3 / e2e_steps}
        # the paper's Table V split (input / kernel / output time), measured one phase at a
        # time without overlap: H2D of the reads, ordering + search on the device copy, D2H of the intervals
        if dense:
            ev3 = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
            dwd = torch.empty(nwords, dtype=torch.int64, device=dev)
            outd = torch.empty((Q, 2), dtype=torch.int32, device=dev)
            permd = torch.empty(Q, dtype=torch.int32, device=dev)
            torch.cuda.synchronize()
            ev3[0].record(stream)
            dwd.copy_(dw, non_blocking=True)
            ev3[1].record(stream)
            idx.order(dwd, None, fixed_len=fixed, out=permd, stream=stream, workspace=ws, key_bases=args.order_bases,
                      n_reads=Q)
            idx.match(dwd, None, fixed_len=fixed, out=outd, stream=stream, workspace=ws, order=permd, n_reads=Q)
            ev3[2].record(stream)
            out_h.copy_(outd, non_blocking=True)
            ev3[3].record(stream)
            torch.cuda.synchronize()
            if not torch.equal(outd.cpu(), out.cpu()):
                raise RuntimeError("dense-layout device path disagrees with the strided path")
            line["e2e"]["split_ms"] = {"input": ev3[0].elapsed_time(ev3[1]), "kernel": ev3[1].elapsed_time(ev3[2]),
                                       "output": ev3[2].elapsed_time(ev3[3])}
            # the bound of the end-to-end path: the host->device copy of the reads alone
            sp = line["e2e"]["split_ms"]
            h2d_rate = Q / (sp["input"] * 1e-3)
            line["e2e"]["bound"] = {"kind": "pcie_h2d", "h2d_GBps": h2d / (sp["input"] * 1e-3) / 1e9,
                                    "h2d_only_queries_per_s": h2d_rate,
                                    "frac": line["e2e"]["value"] / world / h2d_rate}
            del dwd, outd, permd

    # ---- CPU baseline: the oracle on a bounded sample (rank 0, N=1 only) ----
    if rank == 0 and world == 1 and not args.no_cpu and not args.partition:
        got_h = out.cpu().numpy().view(np.uint32)
        line["cpu_baseline"] = cpu_baseline(cfg, ref, idx, words_h.numpy().view(np.uint64),
                                            None if fixed else lens_h.numpy().view(np.uint32), got_h,
                                            args.cpu_seconds, args.cpu_sample)
        del got_h

    if rank == 0:
        print(json.dumps(line), flush=True)
    idx.close()
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
