"""Stall samples per CUDA source line for one kernel (ncu cuda,sass view).
usage: python tools/ncu_lines.py report.ncu-rep kernel_regex [N]"""
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
        d = dict(zip(range(len(hdr)), r))
        s = float(r[4] or 0)
        reasons = sorted(((hdr[i][6:], float(r[i])) for i in range(len(hdr))
                          if hdr[i].startswith("stall_") and "Not Issued" not in hdr[i]
                          and r[i].replace(".", "").isdigit() and float(r[i]) > 0), key=lambda x: -x[1])[:2]
        lines.append((s, f"{fname}:{r[0]}", r[1].strip()[:78], reasons, r[7]))
tot = sum(l[0] for l in lines) or 1
print(f"{kern}: {tot:.0f} samples")
for s, loc, src, reasons, inst in sorted(lines, key=lambda l: -l[0])[:n]:
    print(f"{100 * s / tot:5.1f}% {loc:24s} {src:78s} {[(k, int(v)) for k, v in reasons]} inst={inst}")
