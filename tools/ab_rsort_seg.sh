timeout 600 python -m pytest tests/test_gpu_bzip2.py tests/test_gpu_bunzip2.py -q -x -p no:cacheprovider > gpurun_out/seg_tests.log 2>&1; echo RC=$? >> gpurun_out/seg_tests.log
timeout 500 python tools/stress_bzip2.py 400 43 > gpurun_out/seg_stress.log 2>&1
timeout 600 python tools/stress_roundtrip.py 200 47 >> gpurun_out/seg_stress.log 2>&1
for r in 1 2; do
  PCBZ_RSORT_SEG=0 timeout 300 python tools/bench_bzip2.py 100 >> gpurun_out/seg_ab.log 2>&1; echo "^global" >> gpurun_out/seg_ab.log
  PCBZ_RSORT_SEG=1 timeout 300 python tools/bench_bzip2.py 100 >> gpurun_out/seg_ab.log 2>&1; echo "^segmented" >> gpurun_out/seg_ab.log
done
PCBZ_RSORT_SEG=1 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/seg_launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/seg_ncu.log 2>&1
