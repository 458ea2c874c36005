# One `ncu --set full` capture per dominant kernel (after the plain run exits 0):
# config 2 K3, config 4 K3, config 5 K3 + tile kernel, config 5m K3<motion>.
# Writes gpurun_out/roof_<w>.ncu-rep and gpurun_out/roof_<w>_details.csv.
export PYTHONPATH=.
run() {  # workload kernel-regex launch-count
  w=$1; k=$2; c=$3
  timeout 600 ncu --set full --clock-control none --import-source on -k "regex:$k" -s 3 -c $c \
    -f -o gpurun_out/roof_$w python bench.py --workload $w --steps 1 --warmup 3 --no-e2e \
    --no-cpu-baseline --no-secondary > gpurun_out/ncu_full_$w.log 2>&1
  echo ncu_$w=$?
  ncu -i gpurun_out/roof_$w.ncu-rep --page details --csv > gpurun_out/roof_${w}_details.csv 2>/dev/null
}
python bench.py --workload config2 --steps 3 --warmup 3 --no-e2e --no-cpu-baseline --no-secondary \
  > /dev/null 2>&1 && echo plain_ok
run config2 "apply_tma_kernel" 1
run config4 "apply_tma_kernel" 1
run config5 "apply_tma_kernel|tiles_tma_kernel" 2
run config5m "apply_tma_kernel" 1
