cd $GRAFT_REPO_ROOT
for r in 0 1 2; do for w in motion720 motion720gray motion4k; do
  out=$(DF_MOTION_M3_R=$r python bench.py --workload $w --steps 10 --warmup 3 --no-cpu-baseline --no-secondary 2>/dev/null | python -c "import json,sys; d=json.load(sys.stdin); print(d['ms_per_step'], d['roofline']['frac'])")
  echo "default R-index $r $w $out"
done; done
for v in paper_1611_03226_b200/variants/*.so; do for w in motion720 motion720gray motion4k; do
  out=$(DF_CUDA_LIB=$PWD/$v python bench.py --workload $w --steps 10 --warmup 3 --no-cpu-baseline --no-secondary 2>/dev/null | python -c "import json,sys; d=json.load(sys.stdin); print(d['ms_per_step'], d['roofline']['frac'])")
  echo "$(basename $v) $w $out"
done; done
