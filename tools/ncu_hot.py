"""Top SASS instructions by warp-stall samples for one kernel of an ncu report.
usage: python tools/ncu_hot.py report.ncu-rep kernel_regex [N]"""
import csv, io, subprocess, sys

rep, kern = sys.argv[1], sys.argv[2]
n = int(sys.argv[3]) if len(sys.argv) > 3 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--kernel-name", f"regex:{kern}",
                      "--print-source", "sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = rows[1]
data = [r for r in rows[2:] if len(r) == len(hdr) and r[0].startswith("0x")]
si = hdr.index("Warp Stall Sampling (All Samples)")
stall_cols = [i for i, h in enumerate(hdr) if h.startswith("stall_") or "Stall" in h and i > si + 1]
tot = sum(float(r[si] or 0) for r in data)
print(f"{kern}: {len(data)} instructions, {tot:.0f} stall samples")
agg = {}
for i in stall_cols:
    agg[hdr[i]] = sum(float(r[i] or 0) for r in data if r[i].replace('.', '').isdigit())
print("by reason:", sorted(((k, int(v)) for k, v in agg.items() if v), key=lambda x: -x[1])[:10])
for r in sorted(data, key=lambda r: -float(r[si] or 0))[:n]:
    top = sorted(((hdr[i], float(r[i])) for i in stall_cols if r[i].replace('.', '').isdigit() and float(r[i]) > 0),
                 key=lambda x: -x[1])[:3]
    print(f"{float(r[si]):7.0f} {r[0][-5:]} {r[1].strip()[:60]:60s} {top}")
