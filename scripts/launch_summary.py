"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv)."""
import collections, csv, sys

def main(path, title):
    rows = [r for r in csv.reader(open(path)) if len(r) >= 15 and r[12] == "gpu__time_duration.sum"]
    scale = {"ns": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0, "msecond": 1.0, "nsecond": 1e-6}
    tot, cnt = collections.Counter(), collections.Counter()
    for r in rows:
        name = r[4].split("(")[0].split("::")[-1]
        tot[name] += float(r[14].replace(",", "")) * scale.get(r[13], 1e-6)
        cnt[name] += 1
    s = sum(tot.values())
    print(f"# {title}")
    print(f"# total {s:.1f} ms device time over {sum(cnt.values())} launches (cold-cache, serialised: compare shares)")
    for k, v in tot.most_common():
        print(f"{k:32s} {v:10.3f} ms  {100 * v / s:5.1f}%  {cnt[k]:6d} launches")

if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else sys.argv[1])
