"""From an ncu launch list of one epoch (scripts/ncu_round.sh), write the
SpMM DRAM traffic bench.py reports as roofline.traffic:
profiles/ncu_spmm_<config>.json = {dram_bytes_per_epoch, launches, ...}."""
import collections, csv, json, os, sys

path, out = sys.argv[1], sys.argv[2]
rows = list(csv.reader(open(path)))
hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
h, data = rows[hi], rows[hi + 1:]
ki, mi, vi, ui, idi = (h.index(x) for x in ("Kernel Name", "Metric Name", "Metric Value", "Metric Unit", "ID"))
per, names = collections.defaultdict(dict), {}
scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
tscale = {"ns": 1e-9, "nsecond": 1e-9, "us": 1e-6, "usecond": 1e-6, "ms": 1e-3, "msecond": 1e-3}
for r in data:
    v = float(r[vi].replace(",", ""))
    per[r[idi]][r[mi]] = v * (scale.get(r[ui], 1) if "bytes" in r[mi] else tscale.get(r[ui], 1))
    names[r[idi]] = r[ki]
sp = [i for i in per if "spmm" in names[i] and "partition" not in names[i]]
byts = sum(per[i].get("dram__bytes_read.sum", 0) + per[i].get("dram__bytes_write.sum", 0) for i in sp)
secs = sum(per[i].get("gpu__time_duration.sum", 0) for i in sp)
json.dump({"dram_bytes_per_epoch": byts, "spmm_launches": len(sp), "spmm_seconds_serialised": secs,
           "dram_gbs_serialised": byts / secs / 1e9 if secs else None, "source": path,
           "commit": os.environ.get("PK_COMMIT")}, open(out, "w"), indent=1)
print(open(out).read())
