"""Summarise an ncu --metrics gpu__time_duration.sum --csv launch list per kernel."""
import collections
import csv
import re
import sys


def summarise(path, steps=1):
    rows = list(csv.reader(open(path)))
    hdr, data = None, []
    for r in rows:
        if r and r[0] == "ID":
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            data.append(dict(zip(hdr, r)))
    agg = collections.OrderedDict()
    tot = 0.0
    for d in data:
        name = d["Kernel Name"]
        m = re.match(r"(void )?(mp::)?(\w+)(<.*?(SegSched|DenseSched|Split3Sched|ListSched), (mp::)?(\w+))?", name)
        key = (m.group(3) + ("/" + m.group(5) + "/" + m.group(7) if m.group(5) else "")) if m else name[:60]
        key += " grid" + d["Grid Size"]
        v = float(d["Metric Value"].replace(",", ""))
        u = d["Metric Unit"]
        v = v / 1000 if u in ("ns", "nsecond") else (v * 1000 if u in ("ms", "msecond") else v)
        agg.setdefault(key, [0.0, 0])
        agg[key][0] += v
        agg[key][1] += 1
        tot += v
    out = []
    for k, (v, n) in sorted(agg.items(), key=lambda x: -x[1][0]):
        out.append(f"{v / steps:9.1f} us/step {n:4d}x {v / n:8.1f} us/launch {100 * v / tot:5.1f}%  {k}")
    out.append(f"total {tot / steps:.1f} us per step ({len(data)} launches)")
    return "\n".join(out)


if __name__ == "__main__":
    print(summarise(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 1))
