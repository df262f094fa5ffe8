"""Per-kernel share of one bench step from an ncu launch list (--metrics gpu__time_duration.sum --csv).
Kernels of the checksum epilogue after the timed region (torch at:: kernels) are listed apart."""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
h = rows[hi]
ik, iv, iu = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
scale = {"ns": 1e-6, "nsecond": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0, "msecond": 1.0}
tot, cnt, other, acct = collections.Counter(), collections.Counter(), 0.0, 0.0
for r in rows[hi + 1:]:
    if len(r) <= iv:
        continue
    ms = float(r[iv].replace(",", "")) * scale.get(r[iu], 1.0)
    name = r[ik].split("(")[0].replace("void ", "").replace("wasabi::", "").replace("<unnamed>::", "")
    if name.startswith("at::"):
        other += ms
        continue
    if name.startswith("count_acc_kernel"):      # wasabi_row_work / wasabi_count_accumulations: untimed accounting
        acct += ms
        continue
    tot[name] += ms
    cnt[name] += 1
T = sum(tot.values())
print(f"{'kernel':40s} {'launches':>8s} {'ms':>10s} {'share':>7s}")
for k, v in tot.most_common():
    print(f"{k:40s} {cnt[k]:8d} {v:10.3f} {100 * v / T:6.1f}%")
print(f"{'total (our kernels)':40s} {'':8s} {T:10.3f}\n(torch checksum epilogue outside the timed region: {other:.1f} ms; "
      f"count_acc_kernel -- bench's untimed band-work estimate and exact accumulation count: {acct:.1f} ms)")
