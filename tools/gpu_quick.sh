#!/bin/bash
# Iteration session: GPU parity tests, the bench line, one ncu --set full capture.
# Usage: tools/gpu_quick.sh tag [steps] [ncu:0/1]
TAG=${1:-quick}
STEPS=${2:-295}
NCU=${3:-1}
OUT=gpurun_out
mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $OUT/smoke_$TAG.log 2>&1; echo "smoke rc=$?"; tail -2 $OUT/smoke_$TAG.log
timeout 900 python -m pytest tests -q -m gpu -x > $OUT/pytest_gpu_$TAG.log 2>&1; echo "pytest rc=$?"; tail -15 $OUT/pytest_gpu_$TAG.log
timeout 600 python bench.py --steps $STEPS --warmup 5 --no-cpu-baseline > $OUT/bench_$TAG.json 2> $OUT/bench_$TAG.err; echo "bench rc=$?"; tail -c 2500 $OUT/bench_$TAG.json; tail -5 $OUT/bench_$TAG.err
if [ "$NCU" = "1" ]; then
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_(depth_stats|collect|fuse_blocks|retype_place|gc_normals|fallback)" -s 60 -c 12 -o $OUT/prof_$TAG python bench.py --steps 20 --warmup 3 --no-cpu-baseline > $OUT/ncu_full_$TAG.log 2>&1; echo "ncu-full rc=$?"
fi
