"""Summaries of `ncu --page raw --csv` exports (tooling): key metrics per kernel launch,
and DRAM bytes per launch for bench.py's roofline `traffic` (profiles/r02/ncu_traffic.json)."""
import csv, json, sys
KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "lts__t_sector_hit_rate.pct",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "launch__registers_per_thread", "launch__occupancy_limit_registers", "launch__occupancy_limit_shared_mem",
        "smsp__inst_executed.sum", "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_uma.avg.pct_of_peak_sustained_active",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "launch__grid_size", "launch__block_size",
        "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_wait_per_issue_active.ratio"]
UNIT = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-9, "usecond": 1e-6, "msecond": 1e-3,
        "ns": 1e-9, "us": 1e-6, "ms": 1e-3, "B": 1, "KB": 1e3, "MB": 1e6, "GB": 1e9}
def load(path):
    rows = list(csv.reader(open(path)))
    hdr, units = rows[0], rows[1]
    out = []
    for r in rows[2:]:
        d = dict(zip(hdr, r))
        u = dict(zip(hdr, units))
        k = {"kernel": d.get("Kernel Name", "")[:90], "id": d.get("ID")}
        for key in KEYS:
            if key in d and d[key] not in ("", "n/a"):
                try:
                    v = float(d[key].replace(",", ""))
                except ValueError:
                    continue
                k[key] = {"value": v, "unit": u.get(key, "")}
        out.append(k)
    return out
def bytes_of(m):
    return m["value"] * UNIT.get(m["unit"], 1)
if __name__ == "__main__":
    if len(sys.argv) < 2:  # never overwrite the committed traffic file with nothing
        sys.exit("usage: python tools/ncu_summarize.py tag=raw.csv [tag=raw.csv ...]")
    traffic = {}
    for arg in sys.argv[1:]:
        tag, path = arg.split("=")
        ks = load(path)
        json.dump(ks, open(f"profiles/r02/ncu_summary_{tag}.json", "w"), indent=1)
        for k in ks:
            name = "ess_kernel" if "ess_kernel" in k["kernel"] else "ozaki_gemm_kernel" if "ozaki" in k["kernel"] else None
            if name and "dram__bytes_read.sum" in k:
                tot = bytes_of(k["dram__bytes_read.sum"]) + bytes_of(k["dram__bytes_write.sum"])
                traffic.setdefault(tag, {})[name] = {"bytes_per_launch": tot,
                    "read": bytes_of(k["dram__bytes_read.sum"]), "write": bytes_of(k["dram__bytes_write.sum"]),
                    "duration_us": (k["gpu__time_duration.sum"]["value"] * UNIT.get(k["gpu__time_duration.sum"]["unit"], 1e-9) * 1e6
                                    if "gpu__time_duration.sum" in k else None),
                    "source": f"profiles/r02/ncu_summary_{tag}.json (ncu --set full --clock-control none, one launch)"}
    json.dump(traffic, open("profiles/r02/ncu_traffic.json", "w"), indent=1)
    print(json.dumps(traffic, indent=1))
