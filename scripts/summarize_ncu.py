"""Summarize ncu captures into profiles/ (run here, on the CPU box).

    python scripts/summarize_ncu.py REPORT.ncu-rep OUT_PREFIX [--launches N]

Writes OUT_PREFIX.txt (key metrics + top stall lines) and, for a single-launch
capture, OUT_PREFIX.json with dram bytes per launch (used by bench.py's
roofline.traffic)."""
import csv
import io
import json
import subprocess
import sys

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "launch__grid_size",
        "launch__block_size", "launch__registers_per_thread", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_sector_hit_rate.pct",
        "l1tex__t_sector_pipe_lsu_mem_global_op_ld_hit_rate.pct", "smsp__inst_executed.sum",
        "sm__cycles_elapsed.avg.per_second", "launch__shared_mem_per_block_dynamic",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed", "lts__throughput.avg.pct_of_peak_sustained_elapsed",
        "l1tex__throughput.avg.pct_of_peak_sustained_active", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__inst_executed.avg.per_cycle_active",
        "lts__t_sectors.sum", "lts__t_sectors_op_atom.sum", "lts__t_sectors_op_red.sum",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "smsp__warps_eligible.avg.per_cycle_active",
        "launch__occupancy_limit_registers", "sm__maximum_warps_per_active_cycle_pct"]


def ncu(args):
    return subprocess.run(["ncu", "-i"] + args, capture_output=True, text=True, check=True).stdout


def main():
    rep, out = sys.argv[1], sys.argv[2]
    raw = list(csv.reader(io.StringIO(ncu([rep, "--page", "raw", "--csv"]))))
    h, units, v = raw[0], raw[1], raw[2]
    metrics = {k: (v[h.index(k)], units[h.index(k)]) for k in KEYS if k in h}
    name = v[h.index("Kernel Name")] if "Kernel Name" in h else "?"
    src = list(csv.reader(io.StringIO(ncu([rep, "--page", "source", "--csv", "--print-source", "cuda,sass"]))))
    hdr = src[2]
    iS = hdr.index("Warp Stall Sampling (All Samples)")
    stall_cols = [i for i, x in enumerate(hdr) if x.startswith("stall_") and "Not" not in x]
    lines, agg = [], {}
    for r in src[3:]:
        if r and r[0]:
            try:
                st = {hdr[i]: int(r[i]) for i in stall_cols if i < len(r) and r[i].isdigit() and int(r[i]) > 0}
                lines.append((int(r[iS]), r[0], r[1].strip()[:100], st))
                for k, x in st.items():
                    agg[k] = agg.get(k, 0) + x
            except (ValueError, IndexError):
                pass
    # memory traffic per source line: the L2 sector columns of the source page
    sec_cols = [i for i, x in enumerate(hdr) if "Sectors" in x or "Requests" in x]
    sec_rows = []
    for r in src[3:]:
        if r and r[0]:
            vals = {}
            for i in sec_cols:
                try:
                    vals[hdr[i]] = float(r[i].replace(",", ""))
                except (ValueError, IndexError):
                    pass
            if any(vals.values()):
                sec_rows.append((r[0], r[1].strip()[:90], vals))
    tot = max(1, sum(x[0] for x in lines))
    with open(out + ".txt", "w") as f:
        f.write(f"kernel: {name}\nreport: {rep}\n\n")
        for k, (val, unit) in metrics.items():
            f.write(f"{k:70s} {val} {unit}\n")
        f.write("\nstall reasons (samples): " + ", ".join(f"{k}={x}" for k, x in sorted(agg.items(), key=lambda y: -y[1])[:8]) + "\n")
        f.write("\ntop source lines by warp-stall samples (engine.cu line numbers):\n")
        for s, ln, txt, st in sorted(lines, reverse=True)[:25]:
            top = ", ".join(f"{k}={x}" for k, x in sorted(st.items(), key=lambda y: -y[1])[:2])
            f.write(f"{s:7d} {100 * s / tot:5.1f}%  L{ln:>5}  {txt:100s}  [{top}]\n")
        key = next((hdr[i] for i in sec_cols if hdr[i].startswith("L2 Theoretical Sectors Global")
                    and "Excessive" not in hdr[i]), hdr[sec_cols[0]] if sec_cols else None)
        if key:
            tot_sec = max(1.0, sum(v.get(key, 0.0) for _, _, v in sec_rows))
            f.write(f"\nsector columns on the source page: {[hdr[i] for i in sec_cols]}\n")
            f.write(f"top source lines by '{key}' (total {tot_sec:.4g}):\n")
            for ln, txt, v in sorted(sec_rows, key=lambda y: -y[2].get(key, 0.0))[:25]:
                extra = ", ".join(f"{k.replace('L2 Theoretical Sectors ', '')}={x:.3g}" for k, x in v.items()
                                  if x and k != key)[:120]
                f.write(f"{v.get(key, 0.0):12.4g} {100 * v.get(key, 0.0) / tot_sec:5.1f}%  L{ln:>5}  {txt:90s}  [{extra}]\n")
    if "dram__bytes_read.sum" in metrics:
        def mb(x):
            val, unit = x
            scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(unit, 1)
            return float(val.replace(",", "")) * scale
        d = {"kernel": name, "dram_bytes_per_launch": mb(metrics["dram__bytes_read.sum"]) + mb(metrics["dram__bytes_write.sum"]),
             "duration": metrics.get("gpu__time_duration.sum"), "source": rep,
             "note": "ncu --set full --clock-control none, default cache control (caches flushed before the launch)"}
        with open(out + ".json", "w") as f:
            json.dump(d, f, indent=1)
    print("wrote", out + ".txt")


if __name__ == "__main__":
    main()
