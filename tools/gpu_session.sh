#!/bin/bash
# One GPU session: tests, bench (both arms), ncu launch list + full capture.
# Usage: tools/gpu_session.sh [tag] [steps]
TAG=${1:-r1}
STEPS=${2:-295}
OUT=gpurun_out
mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,driver_version --format=csv > $OUT/gpu_$TAG.txt
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $OUT/smoke_$TAG.log 2>&1; echo "smoke rc=$?"
timeout 900 python -m pytest tests -q -m gpu -x > $OUT/pytest_gpu_$TAG.log 2>&1; echo "pytest rc=$?"; tail -3 $OUT/pytest_gpu_$TAG.log
timeout 600 python bench.py --steps $STEPS --warmup 5 > $OUT/bench_$TAG.json 2> $OUT/bench_$TAG.err; echo "bench rc=$?"; tail -c 3000 $OUT/bench_$TAG.json
timeout 400 python bench.py --impl reference --steps 60 --warmup 5 --ref-budget 60 > $OUT/bench_ref_$TAG.json 2> $OUT/bench_ref_$TAG.err; echo "ref rc=$?"; tail -c 1500 $OUT/bench_ref_$TAG.json
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_" --csv --log-file $OUT/launches_$TAG.csv python bench.py --steps 20 --warmup 3 --no-cpu-baseline > $OUT/ncu_bench_$TAG.log 2>&1; echo "ncu-launch rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_(depth_stats|collect|fuse_blocks|retype_place|gc_normals)" -s 50 -c 10 -o $OUT/prof_$TAG python bench.py --steps 20 --warmup 3 --no-cpu-baseline > $OUT/ncu_full_$TAG.log 2>&1; echo "ncu-full rc=$?"
ls -la $OUT
