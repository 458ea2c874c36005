# usage: abrun.sh "<variants>" "<bench args>" reps
for r in $(seq 1 $3); do for n in $1; do
  CAMX_LIB=variants/libcamx_$n.so timeout 200 python bench.py $2 --no-e2e --no-cpu-baseline --steps 30 > gpurun_out/ab_$n.log 2>&1
  tail -1 gpurun_out/ab_$n.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(\"$n\", d[\"ms_per_step\"], d[\"array_frames_per_sec\"], d[\"roofline\"][\"frac\"])" || tail -3 gpurun_out/ab_$n.log
done; done
