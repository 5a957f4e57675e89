"""Summarise an ncu report: headline metrics, stall reasons, hottest SASS
instructions (python scripts/ncu_hot.py report.ncu-rep [launch_index])."""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
li = int(sys.argv[2]) if len(sys.argv) > 2 else 0
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr, data = rows[0], rows[2:]
want = ["Kernel Name", "launch__grid_size", "launch__registers_per_thread", "gpu__time_duration.sum",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_shared_cycles_active.avg.pct_of_peak_sustained_active",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "lts__t_sector_hit_rate.pct", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum"]
d = data[li]
for w in want:
    if w in hdr:
        print(f"  {w} = {d[hdr.index(w)]}")
stall = [h for h in hdr if h.startswith("smsp__pcsamp_warps_issue_stalled") and not h.endswith("not_issued")]
vals = sorted(((float(d[hdr.index(h)].replace(",", "") or 0), h) for h in stall if d[hdr.index(h)] not in ("", "n/a")),
              reverse=True)[:8]
tot = sum(v for v, _ in vals) or 1
for v, h in vals:
    print(f"  {v / tot * 100:5.1f}%  {h.replace('smsp__pcsamp_warps_issue_stalled_', '')}")
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass", "--launch-skip", str(li),
                      "--launch-count", "1"], capture_output=True, text=True).stdout
srows = list(csv.reader(io.StringIO(src)))
sh, sd = srows[1], srows[2:]
ix = {h: i for i, h in enumerate(sh)}
seen, uniq = set(), []
for r in sd:
    if r[0] not in seen:
        seen.add(r[0])
        uniq.append(r)
f = lambda r, h: float((r[ix[h]] or "0").replace(",", "")) if h in ix else 0.0  # noqa: E731
tot = sum(f(r, "Warp Stall Sampling (All Samples)") for r in uniq) or 1
print("  hottest SASS:")
for r in sorted(uniq, key=lambda r: -f(r, "Warp Stall Sampling (All Samples)"))[:12]:
    print(f"  {f(r, 'Warp Stall Sampling (All Samples)') / tot * 100:5.1f}%  {r[ix['Source']].strip()[:90]}")
