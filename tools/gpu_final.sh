#!/bin/bash
# Evidence tail: the default bench line (with the CPU legs) and per-config evidence.
TAG=${1:-final}
OUT=gpurun_out; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 600 python bench.py > $OUT/bench_${TAG}_default.json 2> $OUT/bench_${TAG}_default.err; echo "default bench rc=$?"
CONFIGS="C3 C4 C5" bash tools/gpu_configs_ncu.sh $TAG
