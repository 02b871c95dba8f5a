#!/bin/bash
# bench lines for the other BASELINE configs (C3 refine, C4 4 mm, C5 multi-room)
TAG=${1:-cfg}
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for C in C3 C4; do
  timeout 900 python bench.py --config $C --steps 295 --warmup 5 --no-cpu-baseline > gpurun_out/bench_${TAG}_$C.json 2> gpurun_out/bench_${TAG}_$C.err; echo "$C rc=$?"
done
timeout 1200 python bench.py --config C5 --steps 995 --warmup 5 --no-cpu-baseline > gpurun_out/bench_${TAG}_C5.json 2> gpurun_out/bench_${TAG}_C5.err; echo "C5 rc=$?"
for C in C3 C4 C5; do python -c "
import json,sys; d=json.loads(open('gpurun_out/bench_${TAG}_$C.json').read().strip().splitlines()[-1])
print('$C', 'value', round(d['value']), 'e2e', round(d['e2e']['value']), 'frac', round(d['roofline']['frac'],3), d['roofline']['kernel'], d['final_state'])"; done
