# usage: ab_k3.sh "variantA variantB ..." reps
export PYTHONPATH=.
for r in $(seq 1 $2); do for n in $1; do
  for w in config2 config4 config5m; do
    CAMX_LIB=variants/libcamx_$n.so timeout 300 python bench.py --workload $w --no-e2e --no-cpu-baseline --steps 30 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$n', '$w', d['ms_per_step'], d['roofline']['k_ms_per_launch'], d['roofline']['frac'], d['clocks']['sm_mhz'], d['clocks']['reasons'])"
  done
done; done
