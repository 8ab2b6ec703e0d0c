"""Per-kernel-class duration and DRAM bytes per launch from ncu launch-list CSVs (diagnostics)."""
import collections
import csv
import sys

for path in sys.argv[1:]:
    rows = list(csv.reader(open(path)))
    hdr, data = None, []
    for r in rows:
        if "Kernel Name" in r:
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            data.append(dict(zip(hdr, r)))
    agg = collections.defaultdict(lambda: collections.defaultdict(float))
    cnt = collections.Counter()
    for d in data:
        k = d["Kernel Name"].split("(")[0].replace("void ", "").replace("mk::", "")[:40]
        v = float(d["Metric Value"].replace(",", ""))
        agg[k][d["Metric Name"]] += v
        if d["Metric Name"] == "gpu__time_duration.sum":
            cnt[k] += 1
    tot_gemm = sum(a["dram__bytes_read.sum"] + a["dram__bytes_write.sum"] for k, a in agg.items() if "gemm" in k)
    print(path, "GEMM DRAM GB %.1f" % (tot_gemm / 1e9))
    for k, a in sorted(agg.items(), key=lambda kv: -kv[1]["gpu__time_duration.sum"])[:8]:
        n = cnt[k]
        print("   %-40s n=%3d avg_us=%8.1f dram_MB=%7.0f" % (k, n, a["gpu__time_duration.sum"] / n / 1e3,
                                                         (a["dram__bytes_read.sum"] + a["dram__bytes_write.sum"]) / n / 1e6))
