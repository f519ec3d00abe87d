# A/B of one knob on bench configs, interleaved repetitions:
#   bash tools/ab_knob.sh <tag> <reps> <knob> "<v0> <v1>" <cfg> [<cfg> ...]
TAG=$1; R=$2; KN=$3; VALS=$4; shift 4
for c in "$@"; do
  for i in $(seq 1 $R); do
    for v in $VALS; do
      python bench.py --config $c --steps 10 --warmup 5 --e2e-steps 0 --no-cpu-baseline --no-digest --no-bf16 \
        --knob $KN=$v > gpurun_out/${TAG}_${c}_${KN}${v}_$i.json 2>/dev/null
    done
  done
done
python - "$TAG" <<'PY'
import glob, json, sys, collections
acc = collections.defaultdict(list)
for f in sorted(glob.glob(f"gpurun_out/{sys.argv[1]}_*.json")):
    try:
        d = json.loads(open(f).read().strip().splitlines()[-1])
    except Exception:
        print(f, "no result"); continue
    key = f.rsplit("_", 1)[0].split("/")[-1]
    acc[key].append((d["ms_per_step"], (d.get("cast") or {}).get("ms_per_step"), d["clocks"]["sm_mhz"]))
for k, v in acc.items():
    print(k, "step", [round(a, 3) for a, _, _ in v], "cast", [round(b, 4) if b else None for _, b, _ in v],
          "mhz", [c for _, _, c in v])
PY
