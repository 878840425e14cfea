"""profiles/traffic.json from one scripts/profile.sh directory: DRAM bytes (read + write) per launch
of the dominant kernels, from their ncu --set full captures (bench.py quotes these as `traffic`).
    python scripts/traffic_json.py profiles/<dir>"""
import csv, json, os, sys

d = sys.argv[1]
out = {"source": f"{d}/{{prefill,decode,decode_cfg4}}_raw.csv (one ncu --set full capture each, --clock-control none)"}
keys = ["gpu__time_duration.sum", "sm__pipe_tc_cycles_active.avg.pct_of_peak_sustained_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
        "lts__t_sector_hit_rate.pct", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed"]
for tag, f in (("prefill", "prefill_raw.csv"), ("decode", "decode_raw.csv"), ("decode_cfg4", "decode_cfg4_raw.csv")):
    path = os.path.join(d, f)
    if not os.path.exists(path):
        continue
    rows = list(csv.reader(open(path)))
    hdr, units, vals = rows[0], rows[1], rows[2]
    m = {h: (v, u) for h, u, v in zip(hdr, units, vals)}

    def num(name):
        v, u = m[name]
        x = float(v.replace(",", ""))
        return x * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(u, 1)
    out[f"{tag}_kernel"] = m["Kernel Name"][0][:60]
    rd, wr = num("dram__bytes_read.sum"), num("dram__bytes_write.sum")
    out[f"{tag}_attention_dram_read"] = rd
    out[f"{tag}_attention_dram_write"] = wr
    out[f"{tag}_attention_dram_bytes"] = rd + wr
    for k in keys:
        if k in m:
            out[f"{tag}_{k}"] = f"{m[k][0]} {m[k][1]}"
json.dump(out, open(os.path.join(os.path.dirname(d.rstrip('/')), "traffic.json"), "w"), indent=1)
print(json.dumps(out, indent=1))
