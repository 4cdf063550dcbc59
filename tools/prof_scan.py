"""Profiling driver: build a config's index with the product path and time lv_search phases."""
import os, sys, time, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, numpy as np, lvgen
from bench import build_index
from paper_2410_22347_b200 import lv
cfg = lvgen.get_config(int(os.environ.get("CFG", "2")))
if os.environ.get("LOW"):
    cfg = cfg.replace(low_dtype=os.environ["LOW"])
reps = int(os.environ.get("REPS", "3"))
data = build_index(cfg, log=lambda *a: print(*a, file=sys.stderr))
ix, Qd = data["ix"], data["Qd"]
for flags in os.environ.get("FLAGS", "0").split(","):
    os.environ["LV_DEBUG_SCAN_FLAGS"] = flags
    mains = []
    for _ in range(reps):
        ids, sc, dbg = lv.lv_search(ix, Qd, cfg.k, cfg.R, timing=True)
        mains.append(dbg["kernel_ms"]["main_scan"])
    print(json.dumps({"cfg": cfg.cfg_id, "low": cfg.low_dtype, "flags": flags, "main_ms": sorted(mains)[len(mains) // 2],
                      "phase_ms": dbg["phase_ms"], "kernel_ms": dbg["kernel_ms"], "slots": dbg["slots"],
                      "units": dbg["units"], "grid": dbg["grid"]}), flush=True)
