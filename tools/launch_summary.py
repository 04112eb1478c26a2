"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv) by kernel (dev tool).
    python tools/launch_summary.py gpurun_out/bench_launches.csv "<header line>" > profiles/....txt
"""
import collections, csv, sys

rows = list(csv.reader(open(sys.argv[1])))
hdr = None
tot, cnt = collections.defaultdict(float), collections.Counter()
for r in rows:
    if "Kernel Name" in r and "Metric Value" in r:
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        d = dict(zip(hdr, r))
        if d["Metric Name"] != "gpu__time_duration.sum":
            continue
        scale = {"ns": 1, "nsecond": 1, "us": 1e3, "usecond": 1e3, "ms": 1e6, "msecond": 1e6}[d["Metric Unit"]]
        k = d["Kernel Name"].split("(")[0][:80]
        tot[k] += float(d["Metric Value"].replace(",", "")) * scale
        cnt[k] += 1
T = sum(tot.values())
g = sum(v for k, v in tot.items() if "gemm_bf16_sm100_pair" in k)
print("# ncu launch list of the bench command (cold-cache, serialised: compare SHARES, not absolutes)")
if len(sys.argv) > 2:
    print("# " + sys.argv[2])
print(f"# total {T / 1e6:.1f} ms over {sum(cnt.values())} launches; stage GEMMs (gemm_bf16_sm100_pair) = "
      f"{100 * g / T:.1f}% of device time")
print("ms,share,launches,us_per_launch,kernel")
for k, v in sorted(tot.items(), key=lambda x: -x[1]):
    print(f"{v / 1e6:.2f},{100 * v / T:.1f}%,{cnt[k]},{v / cnt[k] / 1e3:.1f},{k}")
