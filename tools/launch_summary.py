"""Summarise an ncu --csv launch list (gpu__time_duration.sum) by kernel."""
import collections, csv, io, sys

def load(path):
    lines = [l for l in open(path) if l.startswith('"')]
    rows = list(csv.DictReader(io.StringIO("".join(lines))))
    out = []
    for r in rows:
        if r.get("Metric Name") != "gpu__time_duration.sum":
            continue
        v = float(r["Metric Value"].replace(",", ""))
        u = r["Metric Unit"]
        v = v / 1000 if u in ("ns", "nsecond") else (v * 1000 if u in ("ms", "msecond") else v)
        out.append((r["Kernel Name"], v))
    return out

if __name__ == "__main__":
    rows = load(sys.argv[1])
    skip = int(sys.argv[2]) if len(sys.argv) > 2 else 0
    rows = rows[skip:]
    agg = collections.defaultdict(lambda: [0, 0.0])
    for name, v in rows:
        key = name.split("(")[0][:70]
        agg[key][0] += 1
        agg[key][1] += v
    tot = sum(v[1] for v in agg.values())
    print(f"{len(rows)} launches, total {tot:.1f} us")
    for k, v in sorted(agg.items(), key=lambda x: -x[1][1])[:40]:
        print(f"{v[1]:10.1f} us {100 * v[1] / tot:5.1f}%  n={v[0]:5d}  avg={v[1] / v[0]:8.2f}  {k}")
