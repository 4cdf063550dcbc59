"""Summarise ncu captures into committed evidence under profiles/.

  python tools/ncu_summarize.py --cfg 2 --rep gpurun_out/prof_full_cfg2.ncu-rep \
      --launches gpurun_out/launches_cfg2.csv --tag r01

Writes profiles/<tag>_ncu_cfg<cfg>.json (per captured launch: duration, DRAM bytes, tensor-pipe
and SM throughput, occupancy), profiles/<tag>_launches_cfg<cfg>.json (the launch list of one
lv_search: kernel, ncu duration, share of the step) and updates profiles/ncu_traffic.json (DRAM
bytes per launch of the main scan and of K5, read by bench.py).
"""
import argparse
import csv
import io
import json
import os
import subprocess

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
METRICS = {
    "gpu__time_duration.sum": "duration",
    "dram__bytes_read.sum": "dram_read",
    "dram__bytes_write.sum": "dram_write",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active": "tensor_pipe_active_pct",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed": "sm_throughput_pct",
    "sm__warps_active.avg.pct_of_peak_sustained_active": "warps_active_pct",
    "lts__t_sector_hit_rate.pct": "l2_hit_rate_pct",
    "launch__registers_per_thread": "registers_per_thread",
    "launch__grid_size": "grid",
    "launch__block_size": "block",
    "sm__cycles_elapsed.avg.per_second": "sm_clock",
}
UNIT = {"ms": 1e-3, "us": 1e-6, "usecond": 1e-6, "msecond": 1e-3, "nsecond": 1e-9, "ns": 1e-9, "s": 1.0,
        "byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12, "KB": 1e3, "MB": 1e6, "GB": 1e9,
        "Hz": 1.0, "Khz": 1e3, "Mhz": 1e6, "Ghz": 1e9, "KHz": 1e3, "MHz": 1e6, "GHz": 1e9}


def _kernel(name):
    return name.split("(")[0].replace("void ", "").replace("lv::", "").strip()


def summarize_rep(rep):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    out = []
    for r in rows[2:]:
        d = {"kernel": _kernel(r[hdr.index("Kernel Name")])}
        for m, k in METRICS.items():
            if m not in hdr:
                continue
            i = hdr.index(m)
            try:
                v = float(r[i].replace(",", ""))
            except ValueError:
                continue
            scale = UNIT.get(units[i].strip(), 1.0)
            if k == "duration":
                d["duration_ms"] = round(v * scale * 1e3, 5)
            elif k in ("dram_read", "dram_write"):
                d[k + "_bytes"] = int(v * scale)
            elif k == "sm_clock":
                d["sm_clock_mhz"] = round(v * scale / 1e6, 1)
            else:
                d[k] = round(v, 3)
        out.append(d)
    return out


def summarize_launches(path):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
    h = rows[hi]
    ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    ls = []
    for r in rows[hi + 1:]:
        if len(r) <= vi:
            continue
        ls.append({"kernel": _kernel(r[ki]), "ms": float(r[vi].replace(",", "")) * UNIT.get(r[ui], 1e-9) * 1e3})
    # one lv_search = from the last projection split to the end
    starts = [i for i, x in enumerate(ls) if x["kernel"] in ("k_split3", "k_rows_gemm<float, __nv_bfloat16>")]
    step = ls[starts[-1]:] if starts else ls
    tot = sum(x["ms"] for x in step)
    for x in step:
        x["share"] = round(x["ms"] / tot, 4)
        x["ms"] = round(x["ms"], 5)
    return {"note": "ncu gpu__time_duration.sum, --clock-control none, serialised cold-cache launches: compare shares",
            "step_ms_sum": round(tot, 4), "launches": step}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--cfg", type=int, required=True)
    ap.add_argument("--rep")
    ap.add_argument("--launches")
    ap.add_argument("--tag", default="r01")
    ap.add_argument("--key", default=None, help="ncu_traffic.json key (default cfg<cfg>; e.g. cfg2_i8)")
    ap.add_argument("--out", default=os.path.join(ROOT, "profiles"), help="output directory (on a GPU box: under gpurun_out/)")
    a = ap.parse_args()
    prof = a.out
    os.makedirs(prof, exist_ok=True)
    traffic_path = os.path.join(prof, "ncu_traffic.json")
    seed = traffic_path if os.path.exists(traffic_path) else os.path.join(ROOT, "profiles", "ncu_traffic.json")
    traffic = json.load(open(seed)) if os.path.exists(seed) else {}
    key = a.key or f"cfg{a.cfg}"
    t = traffic.setdefault(key, {})
    if a.rep:
        ks = summarize_rep(a.rep)
        json.dump({"source": os.path.basename(a.rep), "kernels": ks}, open(os.path.join(prof, f"{a.tag}_ncu_{key}.json"), "w"), indent=1)
        scans = [k for k in ks if k["kernel"].startswith("k_score_topr")]
        if scans:
            main_scan = max(scans, key=lambda k: k.get("duration_ms", 0))
            t["main_scan_dram_bytes_per_launch"] = main_scan.get("dram_read_bytes", 0) + main_scan.get("dram_write_bytes", 0)
        rr = [k for k in ks if k["kernel"].startswith("k_rerank_topk")]
        if rr:
            k5 = max(rr, key=lambda k: k.get("duration_ms", 0))
            t["rerank_K5_dram_bytes_per_launch"] = k5.get("dram_read_bytes", 0) + k5.get("dram_write_bytes", 0)
        for k in ks:
            print(k)
    if a.launches:
        s = summarize_launches(a.launches)
        json.dump(s, open(os.path.join(prof, f"{a.tag}_launches_{key}.json"), "w"), indent=1)
        for x in s["launches"]:
            print(x)
    json.dump(traffic, open(traffic_path, "w"), indent=1)


if __name__ == "__main__":
    main()
