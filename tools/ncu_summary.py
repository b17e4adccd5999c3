"""Summarise `ncu --set full` reports into profiles/ncu_*_summary.json.
usage: python tools/ncu_summary.py out.json name=path.ncu-rep [...] [--alg=BYTES] [--dominant=name#i]

--dominant names the kernel whose DRAM read + write bytes become the
top-level "dram_bytes_per_launch" (bench.py's roofline.traffic)."""
import csv
import io
import json
import subprocess
import sys

KEYS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "launch__grid_size",
    "launch__block_size", "launch__registers_per_thread", "launch__occupancy_limit_registers",
    "launch__occupancy_limit_shared_mem", "sm__warps_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
    "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "smsp__inst_executed.sum", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
    "lts__t_sector_hit_rate.pct",
]


def raw(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    res = []
    for r in rows[2:]:
        d = {h: (v + (" " + u if u else "")) for h, v, u in zip(hdr, r, units)}
        res.append(d)
    return res


def to_bytes(v):
    num, _, unit = v.partition(" ")
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}[unit.strip() or "byte"]
    return float(num.replace(",", "")) * scale


def dram_bytes(k):
    return to_bytes(k["dram__bytes_read.sum"]) + to_bytes(k["dram__bytes_write.sum"])


def main():
    out = sys.argv[1]
    alg = None
    dominant = None
    summ = {"what": "ncu --set full --clock-control none, one launch each, config-5 bench workload",
            "kernels": {}}
    for a in sys.argv[2:]:
        if a.startswith("--alg="):
            alg = float(a.split("=", 1)[1])
            continue
        if a.startswith("--dominant="):
            dominant = a.split("=", 1)[1]
            continue
        name, path = a.split("=", 1)
        for i, d in enumerate(raw(path)):
            k = {"kernel": d.get("Kernel Name", "?")}
            for key in KEYS:
                if key in d:
                    k[key] = d[key]
            stalls = {h.replace("smsp__average_warps_issue_stalled_", "").replace(
                "_per_issue_active.ratio", ""): d[h] for h in d
                if h.startswith("smsp__average_warps_issue_stalled_") and h.endswith("per_issue_active.ratio")}
            top = sorted(stalls.items(), key=lambda kv: -float(kv[1].split()[0] or 0))[:6]
            k["top_stalls_per_issue"] = dict(top)
            summ["kernels"][f"{name}#{i}"] = k
    if alg:
        summ["algorithmic_bytes_per_launch"] = alg
    if dominant:
        summ["dominant"] = dominant
        summ["dram_bytes_per_launch"] = dram_bytes(summ["kernels"][dominant])
    json.dump(summ, open(out, "w"), indent=1)
    print(json.dumps(summ, indent=1)[:3000])


if __name__ == "__main__":
    main()
