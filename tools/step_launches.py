"""Prints one step's kernels (between the bench's L2-flush fills) from an ncu launch-list CSV."""
import csv, re, sys
rows = list(csv.reader(open(sys.argv[1])))
which = int(sys.argv[2]) if len(sys.argv) > 2 else 2
hdr = None; seq = []
for r in rows:
    if r and r[0] == "ID": hdr = r; continue
    if hdr and len(r) == len(hdr):
        d = dict(zip(hdr, r))
        if d["Metric Name"] == "gpu__time_duration.sum":
            v = float(d["Metric Value"].replace(",", "")); u = d["Metric Unit"]
            us = v / 1000 if u.startswith("n") else (v * 1000 if u.startswith("m") else v)
            seq.append((re.sub(r"\(.*", "", d["Kernel Name"]).replace("void ", "").replace("mtx::<unnamed>::", "")[:44], us))
idx = [i for i, (k, _) in enumerate(seq) if k.startswith("at::vectorized")]
a, b = idx[which], idx[which + 1]
tot = 0
for k, us in seq[a + 1:b]:
    print("%-46s %8.2f" % (k, us)); tot += us
print("step kernel total", round(tot, 1))
