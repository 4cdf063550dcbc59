"""SM clock / power while lv_search runs back to back for a few seconds (per debug flag)."""
import os, sys, time, subprocess, statistics, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, lvgen
from bench import build_index
from paper_2410_22347_b200 import lv
cfg = lvgen.get_config(int(os.environ.get("CFG", "2")))
data = build_index(cfg, log=lambda *a: None)
ix, Qd = data["ix"], data["Qd"]
for flags in os.environ.get("FLAGS", "0,1").split(","):
    os.environ["LV_DEBUG_SCAN_FLAGS"] = flags
    for _ in range(3):
        lv.lv_search(ix, Qd, cfg.k, cfg.R)
    torch.cuda.synchronize()
    p = subprocess.Popen(["nvidia-smi", "--id=0", "--query-gpu=clocks.sm,power.draw", "--format=csv,noheader,nounits",
                          "-lms", "50"], stdout=subprocess.PIPE, text=True)
    t0 = time.time(); n = 0
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    while time.time() - t0 < 4.0:
        for _ in range(20):
            lv.lv_search(ix, Qd, cfg.k, cfg.R)
        n += 20
        torch.cuda.synchronize()
    e1.record(); torch.cuda.synchronize()
    p.terminate(); out = p.communicate()[0].strip().splitlines()
    sm = [float(x.split(",")[0]) for x in out[5:-2] if x.strip()]
    pw = [float(x.split(",")[1]) for x in out[5:-2] if x.strip()]
    print(json.dumps({"flags": flags, "ms_per_search": e0.elapsed_time(e1) / n, "sm_mhz_median": statistics.median(sm),
                      "power_w_median": statistics.median(pw), "samples": len(sm)}), flush=True)
