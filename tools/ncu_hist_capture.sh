# One ncu --set full capture of the bench's C2 hist launch (the top kernel),
# exported to CSV for tools/ncu_summary.py and tools/hist_traffic_json.py.
set -e
ncu --set full --clock-control none --import-source on -k regex:judge_hist -s 3 -c 1 -f -o gpurun_out/hist_full \
  python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-pipeline > gpurun_out/hist_full.log 2>&1
ncu -i gpurun_out/hist_full.ncu-rep --page raw --csv > gpurun_out/hist_full_raw.csv
ncu -i gpurun_out/hist_full.ncu-rep --page source --csv > gpurun_out/hist_full_source.csv
