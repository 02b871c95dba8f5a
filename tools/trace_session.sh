#!/bin/bash
# per-CTA kernel timelines of two C2 frames + the GPU parity tests + a bench line
TAG=${1:-t}
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 900 python -m pytest tests -q -m gpu -x > gpurun_out/pytest_gpu_$TAG.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu_$TAG.log
python tools/trace_frame.py 40 C2 > gpurun_out/trace_$TAG.txt 2>&1; echo rc=$?
python tools/trace_frame.py 150 C2 >> gpurun_out/trace_$TAG.txt 2>&1; echo rc=$?
cat gpurun_out/trace_$TAG.txt
timeout 600 python bench.py --steps 295 --warmup 5 --no-cpu-baseline > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err; echo "bench rc=$?"
python -c "
import json; d=json.load(open('gpurun_out/bench_$TAG.json'))
print('value', round(d['value']), 'e2e', round(d['e2e']['value']), 'phases', {k: round(v*1e3,1) for k,v in d['phase_ms_mean'].items()}, 'frac', round(d['roofline']['frac'],3))"
