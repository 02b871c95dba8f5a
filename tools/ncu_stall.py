"""Warp-stall samples per CUDA source line for one kernel (ncu source page),
with the dominant stall reasons.  usage: python tools/ncu_stall.py report.ncu-rep kernel_regex [N]"""
import csv, io, subprocess, sys

rep, kern = sys.argv[1], sys.argv[2]
n = int(sys.argv[3]) if len(sys.argv) > 3 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--kernel-name", f"regex:{kern}",
                      "--print-source", "cuda,sass", "--launch-count", "1"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
fname, hdr, lines = "", None, []
for r in rows:
    if r and r[0] == "File Path":
        fname = r[1].split("/")[-1]
    elif r and r[0] == "Line No":
        hdr = r
    elif hdr and len(r) == len(hdr) and r[0] and r[2] == "-":
        si = hdr.index("Warp Stall Sampling (All Samples)")
        reasons = [(hdr[i], float(r[i] or 0)) for i in range(len(hdr))
                   if hdr[i].startswith("stall_") and "Not Issued" not in hdr[i]]
        reasons = sorted(reasons, key=lambda x: -x[1])[:3]
        lines.append((float(r[si] or 0), f"{fname}:{r[0]}", r[1].strip()[:70],
                      " ".join(f"{k[6:]}={v:.0f}" for k, v in reasons if v)))
tot = sum(l[0] for l in lines) or 1
print(f"{kern}: {tot:.0f} stall samples")
for s, loc, src, rs in sorted(lines, key=lambda l: -l[0])[:n]:
    print(f"{100 * s / tot:5.1f}% {loc:22s} {src:70s} {rs}")
