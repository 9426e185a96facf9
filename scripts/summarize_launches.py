"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv) by kernel.

    python scripts/summarize_launches.py gpurun_out/launches.csv "title" > profiles/rNN_launches.md
"""
import collections
import csv
import sys


def main(path, title):
    rows = list(csv.reader(open(path)))
    hdr = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[hdr]
    ki, mi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    tot, cnt = collections.defaultdict(float), collections.Counter()
    for r in rows[hdr + 1:]:
        if len(r) <= mi:
            continue
        v = float(r[mi].replace(",", ""))
        v = v / 1000 if r[ui] in ("ns", "nsecond") else (v * 1000 if r[ui] in ("ms", "msecond") else v)
        name = r[ki].split("(")[0]
        tot[name] += v
        cnt[name] += 1
    T = sum(tot.values())
    print(f"# {title}")
    print("ncu --metrics gpu__time_duration.sum --clock-control none (cold-cache, serialised: compare SHARES)  ")
    print(f"total {T / 1000:.2f} ms over {sum(cnt.values())} launches\n")
    print("| total ms | share | launches | avg us | kernel |\n|---|---|---|---|---|")
    for k, v in sorted(tot.items(), key=lambda x: -x[1]):
        print(f"| {v / 1000:.3f} | {100 * v / T:.1f}% | {cnt[k]} | {v / cnt[k]:.1f} | `{k[:100]}` |")


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else sys.argv[1])
