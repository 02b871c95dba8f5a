#!/bin/bash
# Per-config evidence (BASELINE configs C3 refine, C4 4 mm, C5 multi-room):
# bench lines, ncu launch lists and one ncu --set full capture each.
# Usage: tools/gpu_configs_ncu.sh tag
TAG=${1:-cfg}
OUT=gpurun_out
mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for C in ${CONFIGS:-C3 C4 C5}; do
  ST=295; [ "$C" = "C5" ] && ST=995
  timeout 1200 python bench.py --config $C --steps $ST --warmup 5 --no-cpu-baseline > $OUT/bench_${TAG}_$C.json 2> $OUT/bench_${TAG}_$C.err; echo "$C bench rc=$?"
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_" --csv --log-file $OUT/launches_${TAG}_$C.csv python bench.py --config $C --steps 20 --warmup 3 --no-cpu-baseline > /dev/null 2>&1; echo "$C launches rc=$?"
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_(collect|fuse_blocks|retype_place|gc_normals)" -s 40 -c 4 -o $OUT/prof_${TAG}_$C python bench.py --config $C --steps 20 --warmup 3 --no-cpu-baseline > $OUT/ncu_full_${TAG}_$C.log 2>&1; echo "$C ncu rc=$?"
done
