# usage: ab.sh tag variant1 variant2 ...   ("main" = product library)
tag=$1; shift
for rep in 1 2; do for v in "$@"; do
  if [ $v = main ]; then unset RB_LIB_VARIANT; else export RB_LIB_VARIANT=$v; fi
  python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e $BENCH_ARGS > gpurun_out/${tag}_$v.json 2>gpurun_out/${tag}_$v.err
  python -c "import json;d=json.load(open('gpurun_out/${tag}_$v.json'));r=d['roofline'];print('$v', round(d['ms_per_step'],1), round(r['avg_launch_ms'],3), round(r['frac'],4), d['clocks']['sm_mhz'], d.get('result'))" || tail -3 gpurun_out/${tag}_$v.err
done; done
