"""Summaries of ncu output for profiles/ (run here, on the files gpurun brought back).

    python tools/ncu_summary.py launches <launches.csv> <out.json> [--command "..."]
        per-kernel totals and shares of the superstep kernels from an
        `ncu --metrics gpu__time_duration.sum --csv` launch list (fixture kernels excluded)
    python tools/ncu_summary.py full <report.ncu-rep> <out.json>
        selected metrics of every kernel in an `ncu --set full` report (`ncu -i --page raw`)
"""
import csv
import io
import json
import subprocess
import sys
from collections import OrderedDict

FIXTURE = ("cub::", "DeviceRadixSort", "DeviceSegmentedRadixSort", "(anonymous namespace)",
           "<unnamed>", "at::", "void at::", "rmat", "k_count_slots", "k_fill_coo", "k_scatter",
           # graph create (outside every timed superstep): relabel, derived CSR, plans
           "k_transpose", "k_degree_", "k_relabel_", "k_gather_u32", "k_iota_u32", "k_run_",
           "k_invert_perm", "k_plan_", "k_chunk_", "k_unpack_w", "k_count_nondangling",
           "k_validate", "k_copy_words", "k_noop",
           # the flagged PageRank plan, built once per graph before its first PageRank run
           "k_flag_rows", "k_flag_ranges")

FULL_METRICS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "lts__t_sector_hit_rate.pct", "l1tex__t_sector_hit_rate.pct",
    "lts__throughput.avg.pct_of_peak_sustained_elapsed",
    "l1tex__throughput.avg.pct_of_peak_sustained_active",
    "smsp__inst_executed.sum", "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
    "launch__grid_size", "launch__block_size", "lts__t_sectors_srcunit_tex_op_read.sum",
    "lts__t_requests_srcunit_tex_op_read.sum",
    "l1tex__m_l1tex2xbar_req_cycles_active.avg.pct_of_peak_sustained_elapsed",
    "lts__t_tag_requests.avg.pct_of_peak_sustained_elapsed",
    "l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed",
]


def _rows(text):
    lines = [ln for ln in text.splitlines() if ln.startswith('"')]
    return list(csv.DictReader(io.StringIO("\n".join(lines))))


def launches(path, out, command=None):
    rows = _rows(open(path).read())
    per = OrderedDict()
    units = set()
    for r in rows:
        if r.get("Metric Name") != "gpu__time_duration.sum":
            continue
        name = r["Kernel Name"]
        unit = r.get("Metric Unit", "")
        units.add(unit)
        v = float(r["Metric Value"].replace(",", ""))
        scale = {"ns": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0, "msecond": 1.0,
                 "nsecond": 1e-6}.get(unit, 1e-6)
        ms = v * scale
        if any(f in name for f in FIXTURE):
            continue
        short = name.split("(")[0]
        d = per.setdefault(short, {"kernel": short, "launches": 0, "total_ms": 0.0})
        d["launches"] += 1
        d["total_ms"] += ms
    total = sum(d["total_ms"] for d in per.values())
    ks = sorted(per.values(), key=lambda d: -d["total_ms"])
    for d in ks:
        d["mean_ms"] = d["total_ms"] / d["launches"]
        d["share"] = d["total_ms"] / total if total else None
    res = {"command": command, "units_seen": sorted(units),
           "note": "cold-cache, serialised per-launch times: compare SHARES, not absolutes. "
                   "Fixture kernels (graph generation/sort) excluded from the share table.",
           "superstep_kernels_total_ms": total, "superstep_kernels": ks}
    json.dump(res, open(out, "w"), indent=1)
    for d in ks[:12]:
        print(f"{d['share']:.3f} {d['launches']:5d} {d['mean_ms']:8.3f} ms  {d['kernel']}")


def full(rep, out):
    text = subprocess.check_output(["ncu", "-i", rep, "--page", "raw", "--csv"], text=True)
    rows = list(csv.reader(io.StringIO(text)))
    head, units, data = rows[0], rows[1], rows[2:]
    res = []
    for r in data:
        rec = {"kernel": r[head.index("Kernel Name")], "id": r[head.index("ID")], "metrics": {}}
        for m in FULL_METRICS:
            if m in head:
                i = head.index(m)
                rec["metrics"][m] = {"value": r[i], "unit": units[i]}
        res.append(rec)
    json.dump(res, open(out, "w"), indent=1)
    for rec in res:
        mm = rec["metrics"]
        print(rec["kernel"][:70], {k.split("__")[1][:30]: v["value"] for k, v in mm.items()})


if __name__ == "__main__":
    if sys.argv[1] == "launches":
        cmd = sys.argv[sys.argv.index("--command") + 1] if "--command" in sys.argv else None
        launches(sys.argv[2], sys.argv[3], cmd)
    else:
        full(sys.argv[2], sys.argv[3])
