"""Summarise an ncu --set full capture and a launch-list CSV into profiles/.
usage: python tools/ncu_summary.py TAG report.ncu-rep launches.csv bench.json [CONFIG]
writes profiles/TAG_summary.md and refreshes profiles/ncu_traffic.json (the
per-launch DRAM bytes bench.py reports as roofline.traffic, per BASELINE config;
CONFIG defaults to C2)."""
import csv
import io
import json
import statistics
import subprocess
import sys
from pathlib import Path

tag, rep, launches, bench = sys.argv[1:5]
config = sys.argv[5] if len(sys.argv) > 5 else "C2"
ROOT = Path(__file__).resolve().parents[1]
METRICS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
           "lts__t_sector_hit_rate.pct", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
           "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
           "launch__grid_size", "launch__block_size", "smsp__inst_executed.sum",
           "sm__cycles_active.avg", "sm__cycles_elapsed.avg"]
out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv", "--print-units", "base", "--metrics", ",".join(METRICS)],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr, units, data = rows[0], rows[1], rows[2:]
ki = hdr.index("Kernel Name")
per = {}
for r in data:
    k = r[ki].split("(")[0]
    per.setdefault(k, []).append({m: float((r[hdr.index(m)] or "0").replace(",", "")) for m in METRICS})
lines = [f"# {tag}: ncu --set full (cold cache, serialised replay), {config} frames", "",
         "| kernel | launches | time us | DRAM read MB | DRAM write MB | L2 hit % | SM thru % | warps active % | regs | grid x block | warp-inst | SM active/elapsed |",
         "|---|---|---|---|---|---|---|---|---|---|---|---|"]
traffic = {}
for k, L in per.items():
    m = {q: statistics.mean(x[q] for x in L) for q in METRICS}
    traffic[k] = m["dram__bytes_read.sum"] + m["dram__bytes_write.sum"]
    lines.append(f"| {k} | {len(L)} | {m['gpu__time_duration.sum'] / 1e3:.1f} | {m['dram__bytes_read.sum'] / 1e6:.2f} | "
                 f"{m['dram__bytes_write.sum'] / 1e6:.2f} | {m['lts__t_sector_hit_rate.pct']:.1f} | "
                 f"{m['sm__throughput.avg.pct_of_peak_sustained_elapsed']:.1f} | "
                 f"{m['sm__warps_active.avg.pct_of_peak_sustained_active']:.1f} | {m['launch__registers_per_thread']:.0f} | "
                 f"{m['launch__grid_size']:.0f} x {m['launch__block_size']:.0f} | {m['smsp__inst_executed.sum'] / 1e6:.2f}M | "
                 f"{m['sm__cycles_active.avg'] / max(m['sm__cycles_elapsed.avg'], 1):.2f} |")
# launch list (gpu__time_duration per launch)
lt = {}
txt = Path(launches).read_text().splitlines()
start = next(i for i, l in enumerate(txt) if l.startswith('"ID"'))
for r in csv.DictReader(txt[start:]):
    if r.get("Metric Name") == "gpu__time_duration.sum":
        lt.setdefault(r["Kernel Name"].split("(")[0], []).append(float(r["Metric Value"].replace(",", "")))
lines += ["", "Launch list (`ncu --metrics gpu__time_duration.sum --clock-control none`, every launch of the run):", "",
          "| kernel | launches | mean us | share of frame |", "|---|---|---|---|"]
lt.pop("k_norm_bounds", None)   # once per intrinsics (engine setup), not a frame kernel
tot = sum(sum(v) for v in lt.values())
for k, v in sorted(lt.items(), key=lambda kv: -sum(kv[1])):
    lines.append(f"| {k} | {len(v)} | {statistics.mean(v) / 1e3:.1f} | {sum(v) / tot:.2f} |")
b = json.loads(Path(bench).read_text().strip().splitlines()[-1])
lines += ["", f"bench (same code): value {b['value']:.0f} frames/s ({b['ms_per_step'] * 1e3:.1f} us/frame), "
              f"e2e {b['e2e']['value']:.0f} frames/s, roofline {b['roofline']['kernel']} "
              f"{b['roofline']['achieved']:.0f} GB/s = {100 * b['roofline']['frac']:.1f}% of {b['roofline']['peak']:.0f} GB/s, "
              f"frame {100 * b['roofline']['frame_frac']:.1f}%; phases (profiled pass, ms) {json.dumps({k: round(v, 4) for k, v in b['phase_ms_mean'].items()})}"]
(ROOT / "profiles" / f"{tag}_summary.md").write_text("\n".join(lines) + "\n")
tp = ROOT / "profiles" / "ncu_traffic.json"
tj = json.loads(tp.read_text()) if tp.exists() else {}
tj.setdefault("by_config", {})[config] = traffic
tj.setdefault("sources", {})[config] = f"profiles/{tag}_summary.md (ncu --set full, {config} frames, per launch)"
if config == "C2":
    tj["source"] = tj["sources"]["C2"]
    tj["dram_bytes_per_launch"] = traffic
tp.write_text(json.dumps(tj, indent=1))
print("\n".join(lines))
