#!/bin/bash
# One iteration on the box: GPU tests of the in-tree build, then an A/B of the
# stream period against a baseline build, then the bench line.
# Usage: tools/gpu_ab.sh tag [pytest-args]
TAG=${1:-ab}; shift
OUT=gpurun_out; mkdir -p $OUT
timeout 900 python -m pytest tests -q -m gpu -x ${@} > $OUT/pytest_gpu_$TAG.log 2>&1; echo "pytest rc=$?"; tail -4 $OUT/pytest_gpu_$TAG.log
timeout 600 bash tools/ab_stream.sh 3 ${AB_LIBS:-ab/libA.so ab/libB.so} > $OUT/ab_$TAG.log 2>&1; cat $OUT/ab_$TAG.log
timeout 600 python bench.py --steps 295 --warmup 5 --no-cpu-baseline > $OUT/bench_$TAG.json 2> $OUT/bench_$TAG.err; echo "bench rc=$?"; python -c "
import json;d=json.load(open('$OUT/bench_$TAG.json'));print({k:d[k] for k in ('value','ms_per_step')}, d['value_l2_flushed']['value'], d['e2e']['value'], d['roofline']['frac'], d['phase_ms_mean'], d.get('resumes_in_timed_region'), d.get('overlapped_frames'))"
