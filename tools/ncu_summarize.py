"""Summarise ncu outputs into profiles/ (run in the build container).

    python tools/ncu_summarize.py --launches gpurun_out/launches.csv \
        --rep gpurun_out/prof.ncu-rep --tag r01

Writes profiles/<tag>_launches.csv (per-kernel share of device time) and
profiles/ncu_summary.json (DRAM traffic per launch of the profiled kernels,
read by bench.py as roofline.traffic).
"""
import argparse
import collections
import csv
import json
import subprocess
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent


def launches(path: Path):
    rows = list(csv.reader(path.open()))
    hdr = None
    out = []
    for r in rows:
        if "Kernel Name" in r:
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            d = dict(zip(hdr, r))
            if d.get("Metric Name") == "gpu__time_duration.sum":
                out.append((d["Kernel Name"], float(d["Metric Value"])))
    return out


def raw_metrics(rep: Path):
    if rep.suffix == ".csv":  # `ncu -i rep --page raw --csv` already run on the GPU box (reports can exceed the copy-back limit)
        txt = rep.read_text()
    else:
        txt = subprocess.run(["ncu", "-i", str(rep), "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(txt.splitlines()))
    hdr, units = rows[0], rows[1]
    res = []
    for r in rows[2:]:
        d = dict(zip(hdr, r))
        res.append(d)
    return res, dict(zip(hdr, units))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--launches")
    ap.add_argument("--rep")
    ap.add_argument("--tag", default="r01")
    ap.add_argument("--no-shares", action="store_true", help="do not replace launch_shares in ncu_summary.json")
    a = ap.parse_args()
    prof = ROOT / "profiles"
    prof.mkdir(exist_ok=True)
    summary_path = prof / "ncu_summary.json"
    summary = json.loads(summary_path.read_text()) if summary_path.exists() else {}
    if a.launches:
        ls = launches(Path(a.launches))
        tot = collections.defaultdict(float)
        cnt = collections.Counter()
        for name, ns in ls:
            key = name.split("(")[0].replace("void ", "")
            tot[key] += ns
            cnt[key] += 1
        allns = sum(tot.values())
        out = prof / f"{a.tag}_launches.csv"
        with out.open("w") as f:
            w = csv.writer(f)
            w.writerow(["kernel", "launches", "total_us", "mean_us", "share"])
            for k in sorted(tot, key=lambda k: -tot[k]):
                w.writerow([k, cnt[k], f"{tot[k] / 1e3:.1f}", f"{tot[k] / cnt[k] / 1e3:.2f}", f"{tot[k] / allns:.4f}"])
        if not a.no_shares:
            summary["launch_shares"] = {k: tot[k] / allns for k in tot}
        print(out.read_text())
    if a.rep:
        recs, units = raw_metrics(Path(a.rep))
        per = {}
        for d in recs:
            name = d.get("Kernel Name", "?").split("(")[0].replace("void ", "")
            rb = float(d.get("dram__bytes_read.sum", "nan") or "nan")
            wb = float(d.get("dram__bytes_write.sum", "nan") or "nan")
            scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
            rb *= scale.get(units.get("dram__bytes_read.sum", "byte"), 1)
            wb *= scale.get(units.get("dram__bytes_write.sum", "byte"), 1)
            t = float(d.get("gpu__time_duration.sum", "nan") or "nan")
            tu = units.get("gpu__time_duration.sum", "nsecond")
            t_us = t * {"nsecond": 1e-3, "usecond": 1.0, "msecond": 1e3, "ms": 1e3, "us": 1.0,
                        "ns": 1e-3}.get(tu, 1.0)
            fp64 = d.get("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active")
            dmma = d.get("sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active")
            dram = d.get("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed")
            per.setdefault(name, []).append({"dram_bytes": rb + wb, "duration_us": t_us,
                                             "fp64_pipe_pct": float(fp64) if fp64 else None,
                                             "dmma_pipe_pct": float(dmma) if dmma else None,
                                             "dram_pct": float(dram) if dram else None})
        summary.setdefault("full_capture", {}).update(per)  # merge: one rep per kernel group
        for name, lst in per.items():
            if name.startswith("sample_poly") and "reduce" not in name:
                summary["sample_poly_dram_bytes"] = lst[0]["dram_bytes"]
        print(json.dumps(per, indent=1))
    summary_path.write_text(json.dumps(summary, indent=1))


if __name__ == "__main__":
    main()
