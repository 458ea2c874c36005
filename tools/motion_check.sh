export PYTHONPATH=.
timeout 300 python -m pytest tests/test_gpu_motion.py -x -q 2>&1 | tail -2
timeout 300 python bench.py --workload config5m --no-e2e --no-cpu-baseline --steps 20 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['array_frames_per_sec'], d['roofline']['k_ms_per_launch'], d['roofline']['frac'])"
ncu --metrics gpu__time_duration.sum,smsp__inst_executed.sum -k regex:"apply_tma_kernel" --launch-skip 1 -c 1 python tools/roofline_probe.py config5m 2>&1 | grep -E "duration|inst_executed"
