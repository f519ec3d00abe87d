# Same-box A/B of two builds of the library: _old_lib.so (pushed beside the tree) against the tree's
# libfp8train.so, alternated R times; each run's command is "$@" with {tag} replaced by old / new and {r} by the
# repetition.  usage: bash tools/ab_lib.sh R 'python tools/layer_breakdown.py c3 10 > gpurun_out/x_{tag}_{r}.txt'
R=$1; shift
CMD="$*"
L=paper_2507_16099_b200/libfp8train.so
cp $L /tmp/_new_lib.so
for r in $(seq 1 $R); do
  for tag in ${ORDER:-new old}; do
    if [ $tag = old ]; then cp _old_lib.so $L; else cp /tmp/_new_lib.so $L; fi
    c=${CMD//\{tag\}/$tag}; c=${c//\{r\}/$r}
    bash -c "$c"
  done
done
cp /tmp/_new_lib.so $L
