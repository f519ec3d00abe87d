# Repeated bench runs for A/B comparisons: bash tools/rep_bench.sh <tag> <reps> <cfg> [bench args...]
TAG=$1; R=$2; CFG=$3; shift 3
for i in $(seq 1 $R); do
  python bench.py --config $CFG --steps 20 --warmup 5 --e2e-steps 0 --no-cpu-baseline --no-digest "$@" > gpurun_out/${TAG}_${CFG}_$i.json 2>/dev/null
done
