"""Summarise a profile directory (scripts/profile.sh output) into key metrics + launch shares."""
import csv, json, sys, collections

d = sys.argv[1]
out = {}
for k in ("prefill", "decode", "relayout"):
    rows = list(csv.reader(open(f"{d}/{k}_raw.csv")))
    hdr, units, vals = rows[0], rows[1], rows[2]
    m = {h: (v, u) for h, u, v in zip(hdr, units, vals)}
    def g(name):
        v, u = m.get(name, (None, None))
        try:
            return float(v.replace(",", "")), u
        except Exception:
            return None, u
    rec = {"kernel": m.get("Kernel Name", ("", ""))[0][:90]}
    for name in ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
                 "sm__cycles_active.avg", "smsp__issue_active.avg.pct_of_peak_sustained_active",
                 "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
                 "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
                 "dram__throughput.avg.pct_of_peak_sustained_elapsed",
                 "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio"]:
        rec[name] = g(name)
    out[k] = rec
# launch list
rows = list(csv.reader(open(f"{d}/launches.csv")))
hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
hdr = rows[hi]
ik, im, iv, iid = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value"), hdr.index("ID")
launch = collections.OrderedDict()
for r in rows[hi + 1:]:
    key = (int(r[iid]), r[ik].split("(")[0])
    launch.setdefault(key, {})[r[im]] = float(r[iv].replace(",", ""))
out["launches"] = [{"id": k[0], "kernel": k[1], **v} for k, v in launch.items() if "pi::" in k[1]]
json.dump(out, open(f"{d}/summary.json", "w"), indent=1)
for k in ("prefill", "decode", "relayout"):
    print(k, {kk: vv for kk, vv in out[k].items()})
for L in out["launches"]:
    print(L)
