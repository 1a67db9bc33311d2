"""Summarise ncu outputs into profiles/ (run in the build container).

  python tools/summarize_ncu.py --launches gpurun_out/r1_launches.csv \
      --full gpurun_out/r1_full.ncu-rep --tag r1 --config cfg3

Writes profiles/<tag>_launches_<config>.md (per-kernel share of the step from
the `gpu__time_duration.sum` launch list -- cold-cache, serialised, so only
the SHARES are meaningful), profiles/<tag>_full_<config>.md (key `--set full`
metrics per captured launch) and profiles/gemm_traffic.json (DRAM bytes per
GEMM launch, averaged over one layer's GEMM mix -- bench.py's
roofline.traffic).
"""

from __future__ import annotations

import argparse
import collections
import csv
import json
import os
import subprocess

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def short(name: str) -> str:
    base = name.split("(")[0].replace("void ", "")
    return base[:60]


def launches(path: str):
    rows = list(csv.reader(open(path)))
    hdr, out = None, []
    for r in rows:
        if r and r[0] == "ID":
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            d = dict(zip(hdr, r))
            if d["Metric Name"] != "gpu__time_duration.sum":
                continue
            v = float(d["Metric Value"].replace(",", ""))
            unit = d["Metric Unit"]
            us = v / 1e3 if unit in ("ns", "nsecond") else (v if unit in ("us", "usecond") else v * 1e3)
            out.append((short(d["Kernel Name"]), d["Grid Size"], us))
    return out


def full_metrics(path: str):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(raw.splitlines()))
    hdr, units, data = rows[0], rows[1], rows[2:]
    ci = {h: i for i, h in enumerate(hdr)}
    keys = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
            "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
            "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
            "sm__cycles_elapsed.avg.per_second", "launch__registers_per_thread",
            "sm__warps_active.avg.pct_of_peak_sustained_active"]
    out = []
    for d in data:
        rec = {"kernel": short(d[ci["Kernel Name"]]), "grid": d[ci["Grid Size"]]}
        for k in keys:
            if k in ci:
                rec[k] = (d[ci[k]], units[ci[k]])
        out.append(rec)
    return out


def to_bytes(v, unit):
    v = float(v.replace(",", ""))
    return v * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}.get(unit, 1)


def main():
    p = argparse.ArgumentParser()
    p.add_argument("--launches")
    p.add_argument("--full")
    p.add_argument("--tag", default="r1")
    p.add_argument("--config", default="cfg3")
    p.add_argument("--ticks", type=int, default=3)
    a = p.parse_args()
    prof = os.path.join(ROOT, "profiles")
    os.makedirs(prof, exist_ok=True)
    if a.launches:
        ls = launches(a.launches)
        agg = collections.defaultdict(lambda: [0, 0.0])
        for name, grid, us in ls:
            agg[name][0] += 1
            agg[name][1] += us
        tot = sum(v[1] for v in agg.values())
        lines = [f"# {a.tag} launch list, {a.config} ({a.ticks} ticks incl. warm-up)", "",
                 "ncu `--metrics gpu__time_duration.sum --clock-control none`: cold-cache,",
                 "serialised launches -- compare shares, not absolute times.", "",
                 "| kernel | launches | total ms | share |", "|---|---|---|---|"]
        for k, (n, us) in sorted(agg.items(), key=lambda x: -x[1][1]):
            lines.append(f"| `{k}` | {n} | {us / 1e3:.3f} | {100 * us / tot:.1f}% |")
        open(os.path.join(prof, f"{a.tag}_launches_{a.config}.md"), "w").write(
            "\n".join(lines) + "\n")
    if a.full:
        fm = full_metrics(a.full)
        lines = [f"# {a.tag} ncu --set full, {a.config}", "",
                 "| kernel | grid | time | DRAM read | DRAM write | tensor pipe active | "
                 "DRAM throughput | SM clock | regs |", "|---|---|---|---|---|---|---|---|---|"]
        gemm_bytes = []
        for r in fm:
            g = lambda k: " ".join(r[k]) if k in r else "-"  # noqa: E731
            lines.append(
                f"| `{r['kernel']}` | {r['grid']} | {g('gpu__time_duration.sum')} | "
                f"{g('dram__bytes_read.sum')} | {g('dram__bytes_write.sum')} | "
                f"{g('sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed')} | "
                f"{g('gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed')} | "
                f"{g('sm__cycles_elapsed.avg.per_second')} | "
                f"{g('launch__registers_per_thread')} |")
            if "gemm" in r["kernel"]:
                gemm_bytes.append(to_bytes(*r["dram__bytes_read.sum"]) +
                                  to_bytes(*r["dram__bytes_write.sum"]))
        open(os.path.join(prof, f"{a.tag}_full_{a.config}.md"), "w").write("\n".join(lines) + "\n")
        if gemm_bytes:
            path = os.path.join(prof, "gemm_traffic.json")
            d = json.load(open(path)) if os.path.exists(path) else {}
            d[a.config] = sum(gemm_bytes) / len(gemm_bytes)
            json.dump(d, open(path, "w"), indent=1)


if __name__ == "__main__":
    main()
