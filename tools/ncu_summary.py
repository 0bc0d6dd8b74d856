"""Key metrics per captured launch of an ncu --set full report (text table +
JSON of dram bytes per launch for bench.py's roofline.traffic)."""
import csv, io, json, subprocess, sys
rep, out_txt, out_json, title = sys.argv[1], sys.argv[2], sys.argv[3], sys.argv[4]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
h = rows[0]
want = [("gpu__time_duration.sum", "time_us"), ("dram__bytes_read.sum", "dram_rd"),
        ("dram__bytes_write.sum", "dram_wr"), ("lts__t_sector_hit_rate.pct", "l2_hit%"),
        ("l1tex__t_sector_hit_rate.pct", "l1_hit%"),
        ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm%"),
        ("gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed", "mem%"),
        ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue%"),
        ("sm__warps_active.avg.pct_of_peak_sustained_active", "occ%"),
        ("launch__registers_per_thread", "regs"), ("launch__grid_size", "grid"),
        ("smsp__inst_executed.sum", "warp_inst")]
idx = {k: h.index(k) for k, _ in want if k in h}
ki = h.index("Kernel Name")
units = rows[1]
lines = [f"# {title}", "# " + " ".join(f"{n}" for _, n in want)]
agg = {}
for r in rows[2:]:
    name = r[ki].split("(")[0].replace("void ", "")
    vals = []
    for k, n in want:
        if k not in idx:
            vals.append("-")
            continue
        v = r[idx[k]].replace(",", "")
        u = units[idx[k]]
        try:
            x = float(v)
            if u in ("Kbyte",): x *= 1e3
            if u in ("Mbyte",): x *= 1e6
            if u in ("Gbyte",): x *= 1e9
            if u in ("nsecond", "ns"): x *= 1e-3
            if u in ("msecond", "ms"): x *= 1e3
            vals.append(x)
        except ValueError:
            vals.append(v)
    lines.append(f"{name:28s} " + " ".join(f"{v:.4g}" if isinstance(v, float) else str(v) for v in vals))
    d = dict(zip([n for _, n in want], vals))
    a = agg.setdefault(name, [])
    a.append(d)
open(out_txt, "w").write("\n".join(lines) + "\n")
js = {"source": title}
for name, lst in agg.items():
    base = name.replace("ctk::", "").split("<")[0]
    key = {"k_forward": "forward", "k_back": "back"}.get(base, name)
    dr = [x["dram_rd"] + x["dram_wr"] for x in lst if isinstance(x["dram_rd"], float)]
    tm = [x["time_us"] for x in lst if isinstance(x["time_us"], float)]
    js[key] = {"kernel": name, "launches_captured": len(lst),
               "dram_bytes_per_launch": int(sum(dr) / len(dr)) if dr else None,
               "gpu_time_us": round(sum(tm) / len(tm), 2) if tm else None}
json.dump(js, open(out_json, "w"), indent=1)
print(open(out_txt).read())
