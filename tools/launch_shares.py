"""Per-kernel share of GPU time from an ncu launch list (--metrics gpu__time_duration.sum --csv).
usage: launch_shares.py launches.csv"""
import collections
import csv
import sys

rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 5]
h = rows[0]
ik, im, iu, iv = (h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Unit"),
                  h.index("Metric Value"))
tot, cnt = collections.Counter(), collections.Counter()
for r in rows[1:]:
    if r[im] != "gpu__time_duration.sum":
        continue
    v = float(r[iv].replace(",", ""))
    v *= {"ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3, "nsecond": 1e-3}[r[iu]]
    name = r[ik].split("(")[0].replace("void ", "")
    tot[name] += v
    cnt[name] += 1
T = sum(tot.values())
# the bench step launches each of these once (the validators run only in the untimed per-op leg)
STEP = ("k_len8", "k_transcode<U8Pol", "k_len16", "k_transcode<U16Pol", "k_transcode16", "k_combine")


def in_step(k):
    return any(k == p or k.startswith(p + "<") or (p.endswith("Pol") and k.startswith(p))
               for p in STEP)


S = sum(tot[k] / cnt[k] for k in tot if in_step(k))
print(f"{'kernel':40s} {'launches':>8s} {'total_us':>10s} {'share':>7s} {'avg_us':>9s} {'step_share':>10s}")
for k, v in tot.most_common():
    ss = f"{v / cnt[k] / S:10.3f}" if in_step(k) else f"{'-':>10s}"
    print(f"{k:40s} {cnt[k]:8d} {v:10.1f} {v / T:7.3f} {v / cnt[k]:9.1f} {ss}")
