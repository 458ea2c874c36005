# round-end evidence: GPU tests, default bench line, reference arm, ncu launch lists
export PYTHONPATH=.
python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1; echo tests_rc=$?; tail -2 gpurun_out/gpu_tests.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke_rc=$?
timeout 900 python bench.py > gpurun_out/bench.log 2>gpurun_out/bench.err; echo bench_rc=$?
timeout 600 python bench.py --impl reference > gpurun_out/bench_ref.log 2>&1; echo ref_rc=$?
for w in config2 config5 config5m; do
  ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_$w.csv \
    python bench.py --workload $w --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-secondary > gpurun_out/ncu_launch_$w.log 2>&1; echo launches_$w=$?
done
