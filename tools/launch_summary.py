"""Summarise an ncu launch list (--metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum
--csv) of one bench step into profiles/ncu_summary.json: per-kernel launches, time, share of the step,
DRAM bytes; plus the conv kernel's DRAM bytes per step / per launch (the bench's roofline 'traffic').
usage: python tools/launch_summary.py launches.csv out.json [steps]"""
import csv, json, sys
from collections import defaultdict

rows = list(csv.reader(l for l in open(sys.argv[1]) if not l.startswith("==")))
h = rows[0]
ik, iid, im, iv = h.index("Kernel Name"), h.index("ID"), h.index("Metric Name"), h.index("Metric Value")
per = defaultdict(dict)
for r in rows[1:]:
    if len(r) <= iv:
        continue
    per[r[iid]]["name"] = r[ik].split("(")[0].split("<")[0].replace("void ", "").strip()
    per[r[iid]][r[im]] = float(r[iv].replace(",", ""))
k = defaultdict(lambda: {"launches": 0, "time_us": 0.0, "dram_read_MB": 0.0, "dram_write_MB": 0.0})
for v in per.values():
    e = k[v["name"]]
    e["launches"] += 1
    e["time_us"] += v.get("gpu__time_duration.sum", 0.0) / 1e3
    e["dram_read_MB"] += v.get("dram__bytes_read.sum", 0.0) / 1e6
    e["dram_write_MB"] += v.get("dram__bytes_write.sum", 0.0) / 1e6
tot = sum(e["time_us"] for e in k.values()) or 1.0
for e in k.values():
    e["share"] = e["time_us"] / tot
u = k.get("umma_conv_kernel", {"launches": 0, "dram_read_MB": 0, "dram_write_MB": 0})
umma_bytes = (u["dram_read_MB"] + u["dram_write_MB"]) * 1e6
# the list may cover several steps (tools/profile_step.py STEPS=n): 53 conv launches per step
steps = int(sys.argv[3]) if len(sys.argv) > 3 else max(1, round(u["launches"] / 53))
out = {"source": "ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none, "
                 f"{steps} bench step(s) (tools/profile_step.py with the bench's tuned configs); serialised, cold-cache "
                 "launches: compare shares, not absolutes",
       "steps": steps,
       "kernels": dict(k), "umma_dram_bytes_per_step": umma_bytes / steps,
       "umma_dram_bytes_per_launch": umma_bytes / max(1, u["launches"])}
json.dump(out, open(sys.argv[2], "w"), indent=1)
print(json.dumps(out, indent=1))
