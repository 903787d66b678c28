"""Summarise an ncu --csv launch list: per-kernel count, time share, DRAM bytes (first step of launches)."""
import collections
import csv
import sys


def load(path):
    rows = list(csv.reader(open(path)))
    hi = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
    hdr, data = rows[hi], rows[hi + 1:]
    ki, mi, vi, ii = (hdr.index(k) for k in ("Kernel Name", "Metric Name", "Metric Value", "ID"))
    per, names = collections.defaultdict(dict), {}
    for r in data:
        per[int(r[ii])][r[mi]] = float(r[vi].replace(",", ""))
        names[int(r[ii])] = r[ki].split("(")[0].split("<")[0].replace("void ", "")
    return per, names


def summarize(path, first=None, skip=0):
    per, names = load(path)
    ids = sorted(per)[skip:]
    if first:
        ids = ids[:first]
    tot = collections.defaultdict(lambda: [0, 0.0, 0.0])
    for i in ids:
        t = per[i].get("gpu__time_duration.sum", 0.0)
        b = per[i].get("dram__bytes_read.sum", 0.0) + per[i].get("dram__bytes_write.sum", 0.0)
        tot[names[i]][0] += 1
        tot[names[i]][1] += t
        tot[names[i]][2] += b
    T = sum(v[1] for v in tot.values())
    out = [f"{'kernel':28s} {'n':>5s} {'time_us':>10s} {'share':>6s} {'avg_us':>8s} {'dram_GB':>8s} {'GB/s':>8s}"]
    for n, (c, t, b) in sorted(tot.items(), key=lambda x: -x[1][1]):
        out.append(f"{n:28s} {c:5d} {t/1e3:10.1f} {100*t/T:5.1f}% {t/c/1e3:8.2f} {b/1e9:8.3f} {b/t if t else 0:8.1f}")
    out.append(f"total kernel time {T/1e3:.1f} us over {len(ids)} launches")
    return "\n".join(out)


if __name__ == "__main__":
    print(summarize(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else None,
                    int(sys.argv[3]) if len(sys.argv) > 3 else 0))
