#!/bin/bash
# Round-2 iteration session: smoke, GPU tests, bench line, per-CTA traces, optional ncu capture.
# Usage: tools/gpu_r2.sh TAG [tests:0/1] [ncu:0/1]
TAG=${1:-x}; TESTS=${2:-1}; NCU=${3:-0}
OUT=gpurun_out; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $OUT/smoke_$TAG.log 2>&1; echo "smoke rc=$?"; tail -2 $OUT/smoke_$TAG.log
if [ "$TESTS" = "1" ]; then
timeout 1500 python -m pytest tests -q -m gpu -x > $OUT/pytest_gpu_$TAG.log 2>&1; echo "pytest rc=$?"; tail -4 $OUT/pytest_gpu_$TAG.log
fi
timeout 600 python bench.py --steps 295 --warmup 5 --no-cpu-baseline > $OUT/bench_$TAG.json 2> $OUT/bench_$TAG.err; echo "bench rc=$?"; tail -3 $OUT/bench_$TAG.err
python -c "
import json; d=json.loads(open('$OUT/bench_$TAG.json').read().strip().splitlines()[-1])
print('value', round(d['value']), 'e2e', round(d['e2e']['value']), 'raw', round(d['e2e_raw_u16']['value']), 'phases', {k: round(v*1e3,1) for k,v in d['phase_ms_mean'].items()}, 'frac', round(d['roofline']['frac'],3), d['roofline']['kernel'])"
python -c "import paper_1803_03949_b200.build as b; b.build(trace=True)" > /dev/null 2>&1
timeout 300 python tools/trace_frame.py 40 C2 > $OUT/trace_$TAG.txt 2>&1
timeout 300 python tools/trace_frame.py 150 C2 >> $OUT/trace_$TAG.txt 2>&1; echo "trace rc=$?"
if [ "$NCU" = "1" ]; then
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_(collect|fuse_blocks|retype_place|gc_normals)" -s 60 -c 8 -o $OUT/prof_$TAG python bench.py --steps 20 --warmup 3 --no-cpu-baseline > $OUT/ncu_full_$TAG.log 2>&1; echo "ncu-full rc=$?"
fi
