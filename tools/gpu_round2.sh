export PYTHONPATH=.
python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1; echo tests_rc=$?; tail -3 gpurun_out/gpu_tests.log
timeout 900 python bench.py > gpurun_out/bench.log 2>gpurun_out/bench.err; echo bench_rc=$?
for w in config2 config5 config4; do
  ncu --set full --import-source on --clock-control none -k regex:"apply_tma_kernel|tiles_tma_kernel" --launch-skip 1 -c 2 -o gpurun_out/roof_$w python tools/roofline_probe.py $w > gpurun_out/ncu_$w.log 2>&1; echo ncu_$w=$?
done
