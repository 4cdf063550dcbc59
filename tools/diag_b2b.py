"""Diagnostic: host cost and device time of back-to-back lv_search calls vs synchronised calls."""
import os, sys, time, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, lvgen
from bench import build_index
from paper_2410_22347_b200 import lv
cfg = lvgen.get_config(int(os.environ.get("CFG", "2")))
data = build_index(cfg, log=lambda *a: print(*a, file=sys.stderr))
ix, Qd = data["ix"], data["Qd"]
ids = torch.empty((Qd.shape[0], cfg.k), dtype=torch.int32, device="cuda")
sc = torch.empty((Qd.shape[0], cfg.k), dtype=torch.float32, device="cuda")
for _ in range(3):
    lv.lv_search(ix, Qd, cfg.k, cfg.R, out=(ids, sc))
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
for mode in ["sync_each", "b2b", "sync_each", "b2b"]:
    host = []
    e0.record()
    for _ in range(5):
        t = time.perf_counter()
        lv.lv_search(ix, Qd, cfg.k, cfg.R, out=(ids, sc))
        host.append((time.perf_counter() - t) * 1e3)
        if mode == "sync_each":
            torch.cuda.synchronize()
    e1.record()
    torch.cuda.synchronize()
    print(json.dumps({"mode": mode, "dev_ms_per_call": e0.elapsed_time(e1) / 5, "host_ms": [round(h, 3) for h in host]}), flush=True)
