"""Executed warp-instructions per CUDA source line for one kernel (ncu cuda,sass view).
usage: python tools/ncu_inst.py report.ncu-rep kernel_regex [N]"""
import csv, io, subprocess, sys

rep, kern = sys.argv[1], sys.argv[2]
n = int(sys.argv[3]) if len(sys.argv) > 3 else 25
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
        ii = hdr.index("Instructions Executed")
        lines.append((float(r[ii] or 0), f"{fname}:{r[0]}", r[1].strip()[:90]))
tot = sum(l[0] for l in lines) or 1
print(f"{kern}: {tot:.0f} warp-instructions")
for s, loc, src in sorted(lines, key=lambda l: -l[0])[:n]:
    print(f"{100 * s / tot:5.1f}% {s:10.0f} {loc:24s} {src}")
