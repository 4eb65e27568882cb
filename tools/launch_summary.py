"""Summarise an ncu --metrics gpu__time_duration.sum --csv launch list (last step)."""
import collections, csv, io, sys
path = sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/launches.csv"
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 2
txt = open(path).read()
rows = list(csv.DictReader(io.StringIO(txt[txt.index('"ID"'):])))
rows = [r for r in rows if r.get("Metric Name") == "gpu__time_duration.sum"]
last = rows[len(rows) - len(rows) // steps:]
agg = collections.defaultdict(lambda: [0, 0.0])
for r in last:
    name = r["Kernel Name"].split("(")[0].replace("<unnamed>::", "").replace("(anonymous namespace)::", "")
    agg[name + " " + r["Grid Size"]][0] += 1
    agg[name + " " + r["Grid Size"]][1] += float(r["Metric Value"]) / 1e6
tot = sum(v[1] for v in agg.values())
print(f"total {tot:.3f} ms over {len(last)} launches")
for k, v in sorted(agg.items(), key=lambda x: -x[1][1])[:int(sys.argv[3]) if len(sys.argv) > 3 else 25]:
    print(f"{v[1]:9.3f} ms {v[0]:4d}x {100 * v[1] / tot:5.1f}%  {k[:120]}")
