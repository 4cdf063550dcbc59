#!/usr/bin/env python
"""Benchmark of the lv_search hot path (BASELINE.json metric) — one JSON line on rank 0.

A step = one lv_search call over the config's whole query batch (m = 10 000): K1 projection,
K2/K3 fused reduced scoring + top-R, K4/K5 select + full-D re-rank + top-k.  Inputs are
resident in HBM; X_low and X exceed the 126 MB L2, so the scan streams from HBM every step (no
explicit flush).  Default workload: the largest single-GPU configuration, configs[4] (cfg 5,
GleanVec 10M x 768, C = 32, d = 160, R = 200, k = 10, full vectors fp16); `--config 2` gives the
1M x 512 LeanVec-Sphering line BASELINE.json's metric is also quoted on.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config 2] [--family ood|id]
                  [--impl lv|reference] [--oracle-queries Q] [--no-cpu-baseline]

N > 1 (torchrun): query-sharded replicas — each rank holds the full index and searches its own
m-query batch (weak scaling, no data-path collective).  `--impl reference` times
the CPU oracle (the only reference this paper has) on a bounded query sample per step.  The
index build (fit, K6 encode with its HBM roofline) is reported under `index_build`, outside
the timed step; config 4 has two query families (`--family`), each with its own fit and encode.
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

METRIC = "queries/s and % roofline for reduced-dim scoring+top-R+rerank, 10-recall@10"


def _peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        j = json.load(open(p))
        return {"hbm": j["hbm_gbs"], "bf16": j["bf16_tflops"], "bf16_sus": j.get("bf16_tflops_sustained"),
                "src": "measured (MEASURED_PEAKS.json)"}
    return {"hbm": 6650.0, "bf16": 1590.0, "bf16_sus": 1400.0, "src": "fallback (B200_PROFILING.md)"}


class ClockSampler:
    """nvidia-smi sampling during the timed region (clocks line of B200_PROFILING.md)."""

    def __init__(self, index=0):
        self.index = index
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}",
                 "--query-gpu=clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
                 "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
                 "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap",
                 "--format=csv,noheader,nounits", "-lms", "10"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
            t0 = time.time()
            while not self.lines and time.time() - t0 < 5.0:   # sampler running before the timed region
                time.sleep(0.01)
            self.skip = len(self.lines)
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
                self.proc.wait(timeout=2)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines[getattr(self, "skip", 0):]:
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 8:
                continue
            try:
                sm.append(float(f[0]))
                mx = float(f[1])
            except ValueError:
                continue
            for nm, v in zip(names, f[4:8]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"], "samples": 0}
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": mx, "reasons": sorted(reasons), "samples": len(sm)}


def bind_to_gpu_numa(local_rank, log=print):
    """Pin this process to the CPU cores NVML reports as closest to its GPU, before any pinned host
    buffer is allocated, so the e2e host<->device copies run from the GPU's NUMA node."""
    try:
        import pynvml
        pynvml.nvmlInit()
        h = pynvml.nvmlDeviceGetHandleByIndex(local_rank)
        words = pynvml.nvmlDeviceGetCpuAffinity(h, (os.cpu_count() + 63) // 64)
        cpus = {64 * w + b for w, word in enumerate(words) for b in range(64) if (word >> b) & 1}
        cpus &= set(range(os.cpu_count()))
        if cpus:
            os.sched_setaffinity(0, cpus)
            log(f"[bench] bound to {len(cpus)} CPUs near GPU {local_rank}")
    except Exception as e:   # no NVML / no permission: keep the default placement
        log(f"[bench] NUMA binding skipped: {e}")


def build_index(cfg, rank=0, world=1, log=print, family=None):
    """Generate the config's data, fit with the product path (lv_fit_stats + host eig, GPU k-means
    for GleanVec), encode.  Returns dict with index, device Q, host Q, data."""
    import torch
    import lvgen
    from paper_2410_22347_b200 import fit, lv
    t0 = time.time()
    X = lvgen.database(cfg)
    lo, hi = shard_queries(cfg.m_test, rank, world)
    Q = lvgen.queries(cfg, "test", family=family, m=hi)[lo:hi]
    Ql = lvgen.queries(cfg, "learn", family=family)
    lr = lvgen.learn_rows(cfg)
    log(f"[bench] generated n={cfg.n} D={cfg.D} in {time.time() - t0:.1f}s")
    t0 = time.time()
    Xd = torch.from_numpy(X).cuda()
    Qld = torch.from_numpy(Ql).cuda()
    Xl = Xd[torch.from_numpy(lr).cuda()]
    if cfg.C == 1:
        f = fit.leanvec_sphering_fit(Qld, Xl, cfg.d)
        assign = None
    else:
        f = fit.gleanvec_fit(Qld, Xl, cfg.C, cfg.d, lvgen.kmeanspp_draws(cfg))
        assign = lv.lv_assign_tags(Xd, torch.as_tensor(f["centres"], dtype=torch.float32, device="cuda"))
    torch.cuda.synchronize()
    t_fit = time.time() - t0
    ix = lv.lv_index_create(cfg.D, cfg.d, cfg.C, cfg.low_dtype, cfg.full_dtype,
                            torch.as_tensor(f["A"], dtype=torch.float32), torch.as_tensor(f["B"], dtype=torch.float32))
    torch.cuda.synchronize()
    lv.lv_encode_database(ix, Xd, assign)       # warm (module load, smem attributes); timed below
    torch.cuda.synchronize()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ev0.record()
    lv.lv_encode_database(ix, Xd, assign)
    ev1.record()
    torch.cuda.synchronize()
    t_enc = ev0.elapsed_time(ev1)
    enc_k = lv.lv_encode_timing(ix)
    n_pad = ix.info()["n_pad"]
    log(f"[bench] fit {t_fit:.1f}s encode {t_enc:.1f}ms {enc_k}")
    Qd = torch.from_numpy(Q).cuda()
    del Xd, Xl, Qld
    return {"ix": ix, "Q": Q, "Qd": Qd, "X": X, "A": f["A"], "B": f["B"], "assign": assign,
            "fit_s": t_fit, "encode_ms": t_enc, "encode_kernels": enc_k, "n_pad": n_pad, "gaps": f.get("gaps")}


def _peak_for(cfg):
    """Tensor peak of the scan's dtype: the measured bf16 dense peak, x2 for int8 (the guide's
    nominal ratio, 4.5 vs 2.25 dense P(FL)OP/s)."""
    pk = _peaks()
    f = 2.0 if cfg.low_dtype == "i8" else 1.0
    return pk["bf16"] * f, (pk["bf16_sus"] * f if pk["bf16_sus"] else None), \
        ("int8 dense = 2 x measured bf16 burst (nominal ratio)" if f > 1 else "bf16 dense burst")


def roofline_scan(cfg, ms, m):
    """Dominant kernel: the main k_score_topr launch (every database row x every query, 2 d flop
    per score).  ms = its average launch time over the timed region (CUDA events)."""
    pk = _peaks()
    peak, sus, what = _peak_for(cfg)
    flops = 2.0 * m * cfg.n * cfg.d
    ach = flops / (ms * 1e-3) / 1e12
    return {"bound": "tensor", "achieved": round(ach, 1), "peak": peak, "unit": "TFLOP/s" if cfg.low_dtype != "i8" else "TOP/s",
            "frac": round(ach / peak, 4), "frac_of_sustained": round(ach / sus, 4) if sus else None,
            "peak_source": pk["src"] + ", " + what + " (sustained alongside)",
            "kernel": "k_score_topr main stage (K2/K3 fused scoring + top-R)", "launch_ms": round(ms, 4),
            "algorithmic": f"2*m*n*d = {flops:.3e} flop per launch", "traffic": _ncu_traffic(_tkey(cfg))}


def roofline_rerank(cfg, ms, m):
    """K5 re-rank against HBM.  `frac` uses the DRAM bytes ncu measured for one launch
    (profiles/ncu_traffic.json) when present: candidate rows shared by several queries are partly
    served from L2, so the algorithmic bytes (every candidate's full row once, plus q, candidate ids
    and results) overstate the HBM traffic; their ratio is kept as `algorithmic_frac` (an L2-reuse
    statistic, can exceed 1)."""
    pk = _peaks()
    b = 4 if cfg.full_dtype == "fp32" else 2
    byts = m * cfg.R * cfg.D * b + m * cfg.D * 4 + m * cfg.R * 4 + m * cfg.k * 8
    alg = byts / (ms * 1e-3) / 1e9
    traffic = None
    p = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(p):
        traffic = json.load(open(p)).get(f"cfg{cfg.cfg_id}", {}).get("rerank_K5_dram_bytes_per_launch")   # K5 is the same for every X_low dtype
    ach = traffic / (ms * 1e-3) / 1e9 if traffic else alg
    return {"bound": "hbm", "achieved": round(ach, 1), "peak": pk["hbm"], "unit": "GB/s", "frac": round(ach / pk["hbm"], 4),
            "frac_basis": "ncu DRAM bytes per launch / CUDA-event time" if traffic else "algorithmic bytes (no ncu capture)",
            "kernel": "k_rerank_topk (K5 gather + fp32 dot + top-k)", "launch_ms": round(ms, 4),
            "algorithmic": f"{byts:.3e} B per launch", "algorithmic_frac": round(alg / pk["hbm"], 4), "traffic": traffic}


def scan_phase(cfg, kms, m):
    """The whole scoring + top-R phase (sample stage + threshold select + main scan + K4 top-R
    select) against the bf16 tensor peak, 2 m n d flop (burst; sustained alongside)."""
    peak, sus, _ = _peak_for(cfg)
    ms = kms["sample_stage"] + kms["threshold_select"] + kms["main_scan"] + kms["select_K4"]
    tf = 2.0 * m * cfg.n * cfg.d / (ms * 1e-3) / 1e12
    return {"ms": round(ms, 4), "frac_of_tensor_peak": round(tf / peak, 4),
            "frac_of_sustained": round(tf / sus, 4) if sus else None,
            "note": "sample stage + threshold select + main scan + K4 top-R select (the scoring + top-R phase)"}


def roofline_encode(cfg, k6_ms, n_pad, x_bytes):
    """K6 encode X_low = RNE(B_c x) over the whole database (index build, outside the search step):
    every database row read once (fp32, cfg 5 fp16), every d-wide storage row written once, the
    permutation read once.
    Tensor work: fp32 rows 6 plane products x 2 n d D flop (three-plane bf16 split, lv_proj.cu);
    fp16 rows go in as they are against row-scaled fp16 planes of B: 2 products (bf16 storage) or 3."""
    pk = _peaks()
    byts = cfg.n * cfg.D * x_bytes + n_pad * cfg.d * 2 + n_pad * 4
    note = f"n D {x_bytes} + n_pad d 2 + n_pad 4"
    ach = byts / (k6_ms * 1e-3) / 1e9
    prods = 6 if x_bytes == 4 else (2 if cfg.low_dtype == "bf16" else 3)
    tf = prods * 2.0 * cfg.n * cfg.d * cfg.D / (k6_ms * 1e-3) / 1e12
    return {"bound": "hbm", "achieved": round(ach, 1), "peak": pk["hbm"], "unit": "GB/s", "frac": round(ach / pk["hbm"], 4),
            "tensor_tflops": round(tf, 1), "tensor_frac": round(tf / pk["bf16"], 4),
            "tensor_products": prods,
            "kernel": "k_encode_tc (K6, one persistent launch)", "launch_ms": round(k6_ms, 4),
            "algorithmic": f"{byts:.3e} B per launch ({note})"}


def _tkey(cfg):
    return f"cfg{cfg.cfg_id}" + ("_i8" if cfg.low_dtype == "i8" else "")


def _ncu_traffic(key):
    """dram__bytes_read.sum + dram__bytes_write.sum of the main scan launch, from the committed
    ncu capture summary (profiles/ncu_traffic.json), or None."""
    p = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(p):
        try:
            return json.load(open(p)).get(key, {}).get("main_scan_dram_bytes_per_launch")
        except Exception:
            return None
    return None


def shard_queries(m, rank, world):
    """Query rows [rank * m, (rank + 1) * m) of the config's test stream: each rank searches its own
    batch of the same size (weak scaling, no data-path collective)."""
    return rank * m, (rank + 1) * m


def reduce_max_ms(ms, world):
    """Max over ranks of a per-rank device time (the slowest rank defines the job time)."""
    if world <= 1:
        return ms
    import torch
    import torch.distributed as dist
    dev = "cuda" if dist.get_backend() == "nccl" else "cpu"
    t = torch.tensor([ms], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def oracle_database(cfg, X, B, assign):
    """The oracle's stored reduced database (chunked encode so a 10M x 768 database is never
    converted to fp64 at once): storage-rounded X_low, or for int8 the codes and delta."""
    import oracle as O
    ch = 1 << 19
    chunks = [O.encode(X[lo:lo + ch], B, None if assign is None else assign[lo:lo + ch],
                       store=None if cfg.low_dtype == "i8" else cfg.low_dtype) for lo in range(0, X.shape[0], ch)]
    if cfg.low_dtype != "i8":
        return {"X_low": np.concatenate(chunks)}
    x32 = np.concatenate([c.astype(np.float32) for c in chunks])
    del chunks
    codes, delta = O.quantize_db_i8(x32, assign, cfg.C)
    return {"codes": codes, "delta": delta}


def oracle_search_sample(cfg, Qs, X, A, assign, db):
    """The oracle's search of a query sample against the stored database (project, exhaustive
    reduced top-R, fp64 re-rank, top-k)."""
    import oracle as O
    if cfg.low_dtype == "i8":
        qc, qs = O.quantize_queries_i8(O.project(Qs, A), db["delta"])
        Qeff = qs[:, :, None].astype(np.float64) * qc.astype(np.float64)
        cand, _ = O.reduced_search(Qeff, db["codes"].astype(np.float64), assign, cfg.R, score_fp32=True)
    else:
        cand, _ = O.reduced_search(O.project(Qs, A, store=cfg.low_dtype), db["X_low"], assign, cfg.R)
    ids, _ = O.rerank_topk(Qs, X, cand, cfg.k)
    return ids


def cpu_baseline(cfg, data, nq, log=print):
    """The fp64 oracle (as it stands) on a bounded sample of the same workload."""
    ncores = len(os.sched_getaffinity(0))
    A, B = data["A"], data["B"]
    assign = None if data["assign"] is None else data["assign"].cpu().numpy()
    X = data["X"]
    t0 = time.time()
    db = oracle_database(cfg, X, B, assign)
    t_enc = time.time() - t0
    Qs = data["Q"][:nq]
    t0 = time.time()
    ids = oracle_search_sample(cfg, Qs, X, A, assign, db)
    dt = time.time() - t0
    log(f"[bench] oracle: {nq} queries in {dt:.1f}s (encode {t_enc:.1f}s, untimed)")
    return {"value": round(nq / dt, 3), "unit": "queries/s", "cores": ncores, "kind": "oracle",
            "sample": f"{nq} of {cfg.m_test} queries, full n={cfg.n} database (project + exhaustive reduced top-R + "
                      f"re-rank + top-k, fp64 numpy/OpenBLAS); X_low encode untimed"}, ids, db


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--config", type=int, default=5)
    ap.add_argument("--impl", default="lv", choices=["lv", "reference"])
    ap.add_argument("--oracle-queries", type=int, default=None,
                    help="oracle sample (default 200 queries at 1M rows, 32 at 10M rows)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--family", default=None, help="query family (cfg 4: ood (default) or id; one fit + encode each)")
    ap.add_argument("--low", default=None, choices=["bf16", "fp16", "i8"],
                    help="storage of the reduced vectors (default: the config's; i8 = NEXT-4 8-bit scalar quantisation)")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    log = (lambda *a: print(*a, file=sys.stderr, flush=True)) if rank == 0 else (lambda *a: None)

    import lvgen
    cfg = lvgen.get_config(args.config)
    if args.low:
        cfg = cfg.replace(low_dtype=args.low)
    if args.oracle_queries is None:
        args.oracle_queries = 200 if cfg.n <= 2_000_000 else 32
    family = args.family or cfg.families[-1]
    workload = f"cfg{cfg.cfg_id} {cfg.name}" + (f" [{family} queries]" if len(cfg.families) > 1 else "") + \
        (f" [{cfg.low_dtype} reduced vectors]" if args.low else "")
    conf = {"workload": workload, "n": cfg.n, "D": cfg.D, "d": cfg.d, "C": cfg.C, "m": cfg.m_test, "R": cfg.R,
            "k": cfg.k, "low_dtype": cfg.low_dtype, "full_dtype": cfg.full_dtype,
            "l2": "no flush: X_low and X exceed the 126 MB L2 and are streamed every step"}

    if args.impl == "reference":
        if rank != 0:
            return
        import oracle as O
        X = lvgen.database(cfg)
        Q = lvgen.queries(cfg, "test", family=family)
        Ql = lvgen.queries(cfg, "learn", family=family)
        Xl = X[lvgen.learn_rows(cfg)]
        if cfg.C == 1:
            f = O.sphering_fit(Ql, Xl, cfg.d)
            A, B, assign = f["A"], f["B"], None
        else:
            g = O.gleanvec_fit(Ql, Xl, cfg.C, cfg.d, lvgen.kmeanspp_draws(cfg))
            A, B = g["A"], g["B"]
            assign = np.concatenate([O.assign_tags(X[lo:lo + (1 << 19)], g["centres"])
                                     for lo in range(0, X.shape[0], 1 << 19)])
        db = oracle_database(cfg, X, B, assign)
        per = max(1, args.oracle_queries // (4 if cfg.n <= 2_000_000 else 16))
        def step(i):
            lo = (i * per) % cfg.m_test
            Qs = Q[lo:lo + per]
            oracle_search_sample(cfg, Qs, X, A, assign, db)
        for i in range(args.warmup):
            step(i)
        t0 = time.time()
        for i in range(args.steps):
            step(args.warmup + i)
        dt = time.time() - t0
        v = per * args.steps / dt
        ncores = len(os.sched_getaffinity(0))
        print(json.dumps({"impl": "reference", "metric": METRIC, "value": round(v, 3), "unit": "queries/s",
                          "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
                          "ms_per_step": round(1e3 * dt / args.steps, 3), "higher_is_better": True,
                          "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
                          "config": dict(conf, reference_step=f"{per} queries per step (bounded sample)"),
                          "cpu_baseline": {"value": round(v, 3), "unit": "queries/s", "cores": ncores, "kind": "oracle",
                                           "sample": f"{per} queries per step x {args.steps} steps, full database"},
                          "e2e": {"value": round(v, 3), "unit": "queries/s", "h2d_bytes_per_step": 0,
                                  "d2h_bytes_per_step": 0}}), flush=True)
        return

    import torch
    bind_to_gpu_numa(local, log)
    if world > 1:
        import torch.distributed as dist
        torch.cuda.set_device(local)
        dist.init_process_group("nccl")
    from paper_2410_22347_b200 import lv

    data = build_index(cfg, rank=rank, world=world, log=log, family=family)
    ix, Qd = data["ix"], data["Qd"]
    m = Qd.shape[0]
    ids = torch.empty((m, cfg.k), dtype=torch.int32, device="cuda")
    sc = torch.empty((m, cfg.k), dtype=torch.float32, device="cuda")

    def barrier():
        if world > 1:
            torch.distributed.barrier()

    for _ in range(args.warmup):
        lv.lv_search(ix, Qd, cfg.k, cfg.R, out=(ids, sc))
    torch.cuda.synchronize()
    launches_per_step = lv.lv_search(ix, Qd, cfg.k, cfg.R, out=(ids, sc))[2]["launches"]
    # one untimed pass of the timed loop's shape: the library's event pool then holds the
    # 8 * steps events the timed loop records (no event creation inside the timed region)
    for _ in range(args.steps):
        lv.lv_search(ix, Qd, cfg.k, cfg.R, out=(ids, sc), timing=2)
    torch.cuda.synchronize()
    lv.lv_timing_collect(ix)   # drop anything recorded before the timed region
    st = torch.cuda.current_stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        barrier()
        torch.cuda.synchronize()
        e0.record(st)
        for _ in range(args.steps):
            # timing=2: per-kernel CUDA events on the launch stream, no synchronisation
            lv.lv_search(ix, Qd, cfg.k, cfg.R, out=(ids, sc), timing=2)
        e1.record(st)
        torch.cuda.synchronize()
        barrier()
    ms = reduce_max_ms(e0.elapsed_time(e1), world)
    value = world * m * args.steps / (ms * 1e-3)
    kms, ncalls = lv.lv_timing_collect(ix)   # per-kernel averages over the timed region

    # e2e: public API with HOST buffers (pinned), H2D of Q and D2H of results inside the region
    Qh = torch.from_numpy(data["Q"]).pin_memory()
    ih = torch.empty((m, cfg.k), dtype=torch.int32).pin_memory()
    sh = torch.empty((m, cfg.k), dtype=torch.float32).pin_memory()
    for _ in range(2):
        lv.lv_search_host(ix, Qh, cfg.k, cfg.R, ih, sh)
    barrier()
    torch.cuda.synchronize()
    e0.record(st)
    for _ in range(args.steps):
        lv.lv_search_host(ix, Qh, cfg.k, cfg.R, ih, sh)
    e1.record(st)
    torch.cuda.synchronize()
    ms_e2e = reduce_max_ms(e0.elapsed_time(e1), world)
    barrier()
    if rank != 0:
        torch.distributed.destroy_process_group()
        return

    out = {"metric": METRIC, "value": round(value, 1), "unit": "queries/s", "n_gpus": world, "steps": args.steps,
           "warmup": args.warmup, "ms_per_step": round(ms / args.steps, 4), "higher_is_better": True,
           "scaling": "weak", "vs_baseline": None, "dtype": cfg.low_dtype, "data": "synthetic",
           "config": dict(conf, parallelism=f"query-sharded replicas x{world}" if world > 1 else "single GPU"),
           "kernel_ms": {k: round(v, 4) for k, v in kms.items()},
           "kernel_ms_source": f"CUDA events on the launch stream, average over the {ncalls} timed steps",
           "roofline": roofline_scan(cfg, kms["main_scan"], m),
           "roofline_rerank": roofline_rerank(cfg, kms["rerank_K5"], m),
           "scan_phase": scan_phase(cfg, kms, m),
           "e2e": {"value": round(world * m * args.steps / (ms_e2e * 1e-3), 1), "unit": "queries/s",
                   "h2d_bytes_per_step": int(m * cfg.D * 4), "d2h_bytes_per_step": int(m * cfg.k * 8)},
           "gpu_launches": int(launches_per_step * args.steps),
           "clocks": clk.summary(),
           "index_build": {"fit_s": round(data["fit_s"], 2), "encode_ms": round(data["encode_ms"], 2),
                           "encode_kernels_ms": {k: round(v, 4) for k, v in data["encode_kernels"].items()},
                           "roofline_encode": roofline_encode(cfg, data["encode_kernels"]["encode_K6"], data["n_pad"], data["X"].dtype.itemsize)}}
    if world == 1 and not args.no_cpu_baseline:
        import oracle as O
        nq = min(args.oracle_queries, m)
        cb, ora_ids, _ = cpu_baseline(cfg, data, nq, log=log)
        out["cpu_baseline"] = cb
        gt, _ = O.exact_topk(data["Q"][:nq], data["X"], 10)
        gi = ids[:nq].cpu().numpy().astype(np.int64)
        out["recall_at_10"] = {"gpu": round(O.recall_at_k(gi, gt, 10), 4),
                               "oracle_emulated": round(O.recall_at_k(ora_ids, gt, 10), 4),
                               "sample_queries": nq, "ids_equal_frac": float((gi == ora_ids).all(axis=1).mean())}
    print(json.dumps(out), flush=True)
    if world > 1:
        torch.distributed.destroy_process_group()


if __name__ == "__main__":
    main()
