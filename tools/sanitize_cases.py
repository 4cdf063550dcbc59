"""Small cases of every kernel family, for compute-sanitizer (memcheck / racecheck / synccheck):
the staged path, the sampled path with forced repairs in both unit orders, GleanVec (C = 4), the
int8 scan, the x'-store index with streaming updates, the k-means and statistics kernels, and the
host-buffer entry point.  Prints one line per case; exits non-zero on any library error.

  compute-sanitizer --tool memcheck python tools/sanitize_cases.py
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2410_22347_b200 import fit, lv  # noqa: E402


def data(n, m, D, seed):
    rng = np.random.default_rng(seed)
    X = rng.standard_normal((n, D)).astype(np.float32)
    X /= np.linalg.norm(X, axis=1, keepdims=True)
    Q = rng.standard_normal((m, D)).astype(np.float32)
    Q /= np.linalg.norm(Q, axis=1, keepdims=True)
    return X, Q


def stacks(C, d, D, seed):
    rng = np.random.default_rng(seed)
    return [torch.from_numpy((rng.standard_normal((C, d, D)) / np.sqrt(D)).astype(np.float32)).cuda() for _ in range(2)]


def run(name, low, n, m, D, d, C, R, env=None):
    old = {k: os.environ.get(k) for k in (env or {})}
    os.environ.update(env or {})
    try:
        X, Q = data(n, m, D, n + d)
        A, B = stacks(C, d, D, d)
        ix = lv.lv_index_create(D, d, C, low, "fp32", A, B)
        assign = None if C == 1 else torch.from_numpy(np.random.default_rng(1).integers(0, C, n).astype(np.int32)).cuda()
        lv.lv_encode_database(ix, torch.from_numpy(X).cuda(), assign)
        ids, sc, dbg = lv.lv_search(ix, torch.from_numpy(Q).cuda(), 10, R, cand=True, timing=1)
        torch.cuda.synchronize()
        print(f"{name}: path={dbg['path']} failed={dbg['failed']} launches={dbg['launches']}", flush=True)
    finally:
        for k, v in old.items():
            if v is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = v


def main():
    torch.cuda.set_device(0)
    run("staged bf16", "bf16", 3000, 150, 128, 64, 1, 50)
    run("staged fp16 d=96", "fp16", 2500, 70, 96, 96, 1, 40)
    for dyn in ("1", "0"):
        run(f"sampled+repairs dyn={dyn}", "bf16", 40_000, 200, 128, 32, 1, 64,
            {"LV_SAMPLE_STRIDE": "2", "LV_SAMPLE_GAMMA": "0.2", "LV_DYN_UNITS": dyn})
    run("gleanvec C=4 sampled", "bf16", 40_000, 130, 128, 64, 4, 50, {"LV_SAMPLE_STRIDE": "2"})
    run("int8 staged", "i8", 3000, 140, 128, 96, 1, 50)
    run("int8 sampled+repairs", "i8", 40_000, 130, 128, 64, 1, 64, {"LV_SAMPLE_STRIDE": "2", "LV_SAMPLE_GAMMA": "0.2"})
    # host-buffer entry point (two overlapped batches) and query batching
    X, Q = data(5000, 4200, 64, 7)
    A, B = stacks(1, 32, 64, 7)
    ix = lv.lv_index_create(64, 32, 1, "bf16", "fp32", A, B)
    lv.lv_encode_database(ix, torch.from_numpy(X).cuda())
    lv.lv_search_host(ix, torch.from_numpy(Q).pin_memory(), 10, 50)
    os.environ["LV_MAX_BATCH"] = "1024"
    lv.lv_search(ix, torch.from_numpy(Q).cuda(), 10, 50)
    os.environ.pop("LV_MAX_BATCH")
    torch.cuda.synchronize()
    print("host buffers + batching: ok", flush=True)
    # statistics, k-means kernels
    Xt = torch.from_numpy(X).cuda()
    fit.leanvec_sphering_fit(torch.from_numpy(Q).cuda(), Xt, 32)
    g = fit.gleanvec_fit(torch.from_numpy(Q).cuda(), Xt, 5, 32, np.linspace(0.1, 0.9, 5), max_iter=5)
    print(f"fit + k-means: ok (C={len(g['centres'])})", flush=True)
    # x' store + streaming
    f = fit.flexible_from_stats(*[k[0] if k.ndim == 3 else k for k in lv.lv_fit_stats(torch.from_numpy(Q).cuda(), Xt)],
                                Q.shape[0])
    fx = lv.lv_index_create_flex(64, 32, "bf16", f["A"], f["B"], 20_000)
    lv.lv_encode_database(fx, Xt[:3000])
    lv.lv_stream_observe_queries(fx, torch.from_numpy(Q[:1000]).cuda())
    lv.lv_stream_insert(fx, Xt[3000:4500], np.arange(10_000, 11_500, dtype=np.int32))
    lv.lv_stream_remove(fx, np.concatenate([np.arange(0, 600, 3), np.arange(10_000, 10_300)]).astype(np.int32))
    fit.stream_refresh(fx)
    lv.lv_index_set_search_dim(fx, 32)
    lv.lv_search(fx, torch.from_numpy(Q[:300]).cuda(), 10, 50, cand=True)
    torch.cuda.synchronize()
    print(f"flexible index + streaming: ok (n={fx.info()['n']})", flush=True)


if __name__ == "__main__":
    main()
