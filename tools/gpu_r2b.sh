#!/bin/bash
# Round-2 iteration: named GPU tests first, then the whole GPU suite, the bench line, traces.
# Usage: tools/gpu_r2b.sh TAG "test selection" [full_suite:0/1]
TAG=$1; SEL=$2; FULL=${3:-1}
OUT=gpurun_out; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $OUT/smoke_$TAG.log 2>&1; echo "smoke rc=$?"; tail -2 $OUT/smoke_$TAG.log
if [ -n "$SEL" ]; then
timeout 900 python -m pytest $SEL -q -m gpu -x > $OUT/pytest_sel_$TAG.log 2>&1; echo "sel rc=$?"; tail -30 $OUT/pytest_sel_$TAG.log
fi
timeout 600 python bench.py --steps 295 --warmup 5 --no-cpu-baseline > $OUT/bench_$TAG.json 2> $OUT/bench_$TAG.err; echo "bench rc=$?"; tail -3 $OUT/bench_$TAG.err
python -c "
import json; d=json.loads(open('$OUT/bench_$TAG.json').read().strip().splitlines()[-1])
print('value', round(d['value']), 'flushed', round(d['value_l2_flushed']['value']), 'overlapped', d.get('overlapped_frames'), 'e2e', round(d['e2e']['value']), 'raw', round(d['e2e_raw_u16']['value']), 'phases', {k: round(v*1e3,1) for k,v in d['phase_ms_mean'].items()}, 'frac', round(d['roofline']['frac'],3), d['roofline']['kernel'])"
if [ "$FULL" = "1" ]; then
timeout 1500 python -m pytest tests -q -m gpu -x > $OUT/pytest_gpu_$TAG.log 2>&1; echo "pytest rc=$?"; tail -4 $OUT/pytest_gpu_$TAG.log
fi
