"""Warp-stall breakdown of an ncu --set full capture per SASS region.

    python tools/ncu_stalls.py REPORT.ncu-rep [--from I --to J] [--top N]

Without --from/--to: per-100-instruction buckets (instructions executed,
stall samples). With a range: stall reasons summed over it plus the top
instructions by samples.
"""
import argparse, collections, csv, io, subprocess, sys

ap = argparse.ArgumentParser()
ap.add_argument("report")
ap.add_argument("--from", dest="lo", type=int)
ap.add_argument("--to", dest="hi", type=int)
ap.add_argument("--top", type=int, default=25)
ap.add_argument("--grep", help="print indices of instructions whose text contains this")
a = ap.parse_args()
out = subprocess.run(["ncu", "-i", a.report, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
h, data = rows[1], rows[2:]
isrc, iss, ie = h.index("Source"), h.index("Warp Stall Sampling (All Samples)"), h.index("Instructions Executed")
reasons = [c for c in h if c.startswith("stall_") and "Not Issued" not in c]
n = lambda r, i: int(float(r[i] or 0))
if a.grep:
    for i, r in enumerate(data):
        if a.grep in r[isrc]:
            print(i, n(r, ie), r[isrc][:80])
    sys.exit()
print("total samples", sum(n(r, iss) for r in data), "instructions %.1fM" % (sum(n(r, ie) for r in data) / 1e6))
if a.lo is None:
    b, s = collections.Counter(), collections.Counter()
    for i, r in enumerate(data):
        b[i // 100] += n(r, ie)
        s[i // 100] += n(r, iss)
    for k in sorted(b):
        if b[k] > 1e6 or s[k] > 100:
            print(k * 100, "%.1fM" % (b[k] / 1e6), s[k], data[k * 100][isrc][:60])
    sys.exit()
seg = range(a.lo, a.hi)
agg = collections.Counter()
for i in seg:
    for c in reasons:
        agg[c[6:]] += n(data[i], h.index(c))
print("range samples", sum(n(data[i], iss) for i in seg), "instructions %.1fM" % (sum(n(data[i], ie) for i in seg) / 1e6),
      agg.most_common(8))
for i in sorted(seg, key=lambda i: -n(data[i], iss))[: a.top]:
    r = data[i]
    print(i, n(r, ie), n(r, iss), r[isrc][:64], {c[6:]: r[h.index(c)] for c in reasons if r[h.index(c)] not in ("0", "")})
