"""Per-kernel table from an ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum
CSV (one or more bench steps) -> markdown on stdout; --traffic FILE writes the GEMM class's mean DRAM
bytes per launch (bench.py roofline.traffic)."""
import collections
import csv
import json
import sys


def main():
    path = sys.argv[1]
    rows = list(csv.reader(open(path)))
    hdr, data = None, []
    for r in rows:
        if "Kernel Name" in r:
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            data.append(dict(zip(hdr, r)))
    per = collections.defaultdict(dict)
    for d in data:
        per[(d["ID"], d["Kernel Name"])][d["Metric Name"]] = float(d["Metric Value"].replace(",", ""))
    agg = collections.defaultdict(lambda: [0, 0.0, 0.0])
    for (_, name), m in per.items():
        k = name.split("(")[0].replace("void ", "")
        a = agg[k]
        a[0] += 1
        a[1] += m.get("gpu__time_duration.sum", 0.0) / 1e3
        a[2] += m.get("dram__bytes_read.sum", 0.0) + m.get("dram__bytes_write.sum", 0.0)
    tot = sum(v[1] for v in agg.values())
    print("| kernel | launches | total us | avg us | share | DRAM MB / launch |")
    print("|---|---|---|---|---|---|")
    for k, v in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        print(f"| `{k}` | {v[0]} | {v[1]:.1f} | {v[1] / v[0]:.1f} | {100 * v[1] / tot:.1f}% | {v[2] / v[0] / 1e6:.2f} |")
    print(f"| total | {sum(v[0] for v in agg.values())} | {tot:.1f} | | | |")
    if "--traffic" in sys.argv:
        g = [v for k, v in agg.items() if "gemm_kernel" in k]
        n = sum(v[0] for v in g)
        out = {"dram_bytes_per_launch": sum(v[2] for v in g) / n, "gemm_launches": n,
               "source": path, "note": "mean dram__bytes_read.sum + dram__bytes_write.sum over the GEMM launches "
                                       "of the captured bench steps (ncu serialises kernels; cold-ish L2)"}
        json.dump(out, open(sys.argv[sys.argv.index("--traffic") + 1], "w"), indent=1)


if __name__ == "__main__":
    main()
