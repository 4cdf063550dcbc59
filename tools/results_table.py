"""Markdown results table from the committed bench lines, for DESIGN.md §11.

  python tools/results_table.py --dir profiles/r02        # round 2: bench_cfg<spec>.json per config
  python tools/results_table.py --tag r01                 # round 1: profiles/r01_bench_cfg<N>_v<k>.json
"""
import argparse
import glob
import json
import os

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def latest(tag, c):
    fs = sorted(glob.glob(os.path.join(ROOT, "profiles", f"{tag}_bench_cfg{c}_v*.json")),
                key=lambda p: int(p.rsplit("_v", 1)[1].split(".")[0]))
    return fs[-1] if fs else None


def row(name, f):
    d = json.load(open(f))
    k = d.get("kernel_ms", {})
    r = d.get("roofline", {})
    rr = d.get("roofline_rerank", {})
    ph = d.get("scan_phase", {})
    rec = d.get("recall_at_10", {})
    cb = d.get("cpu_baseline", {})
    re_ = d.get("index_build", {}).get("roofline_encode")
    enc = f"{re_['launch_ms']:.2f} ({re_['frac']:.2f})" if re_ else "-"
    phf = ph.get("frac_of_tensor_peak", ph.get("frac_of_bf16_peak", 0))
    return (f"| {name} | {d['config']['workload']} | {d['value']:,.0f} | {d['e2e']['value']:,.0f} | {d['ms_per_step']:.3f} "
            f"| {k.get('main_scan', 0):.3f} | {r.get('frac', 0):.3f} / {r.get('frac_of_sustained', 0) or 0:.3f} "
            f"| {phf:.3f} | {k.get('rerank_K5', 0):.3f} ({rr.get('frac', 0):.2f}) | {k.get('project_K1', 0):.3f} "
            f"| {k.get('sample_stage', 0) + k.get('threshold_select', 0):.3f} | {k.get('select_K4', 0):.3f} "
            f"| {k.get('repairs', 0):.3f} | {rec.get('gpu', '-')} / {rec.get('oracle_emulated', '-')} "
            f"| {cb.get('value', '-')} ({cb.get('cores', '-')}) | {d['clocks'].get('sm_mhz')} {','.join(d['clocks'].get('reasons', []))} "
            f"| {enc} | {os.path.relpath(f, ROOT)} |")


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--tag", default=None)
    ap.add_argument("--dir", default=None)
    a = ap.parse_args()
    print("| cfg | workload | queries/s | e2e q/s | ms/step | main scan ms | main scan frac of tensor peak (burst / sustained) "
          "| scoring+top-R phase frac | K5 ms (frac of HBM) | K1 | sample+select | K4 | repairs "
          "| recall GPU / emulated oracle | oracle q/s (cores) | SM MHz | K6 encode ms (frac of HBM) | file |")
    print("|---|---|---|---|---|---|---|---|---|---|---|---|---|---|---|---|---|---|")
    if a.dir:
        order = ["5", "2", "3", "1", "4familyood", "4familyid", "2lowi8", "5lowi8"]
        for c in order:
            f = os.path.join(ROOT, a.dir, f"bench_cfg{c}.json")
            if os.path.exists(f):
                print(row(c, f))
        return
    for c in ["1", "2", "3", "4", "4id", "5"]:
        f = latest(a.tag or "r01", c)
        if f:
            print(row(c, f))


if __name__ == "__main__":
    main()
