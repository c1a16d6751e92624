# BWT radix-sort A/B: the current build vs a build whose sort is CUB's
# (paper_2310_09467_b200/_native/variants/libpcbz_cub.so, e.g. made with
#   python tools/build_variants.py --git 3877349 cub && cp .../variants/cub/libpcbz_b200.so .../variants/libpcbz_cub.so
# -- 3877349 is the last commit before csrc/radix_sort.cuh).  Byte-exactness
# tests + stress, two interleaved tools/bench_bzip2.py rounds, and ncu
# launch lists of both (summarised in profiles/r02_rsort_launches_summary.txt).
set -x
rm -f gpurun_out/rsort_ab.log
timeout 600 python -m pytest tests/test_gpu_bzip2.py tests/test_gpu_bunzip2.py -q -x -p no:cacheprovider > gpurun_out/rsort_tests.log 2>&1; echo RC=$? >> gpurun_out/rsort_tests.log
timeout 600 python tools/stress_bzip2.py 200 7 > gpurun_out/rsort_stress.log 2>&1; echo RC=$? >> gpurun_out/rsort_stress.log
for r in 1 2; do
  PCBZ_LIB=paper_2310_09467_b200/_native/variants/libpcbz_cub.so timeout 300 python tools/bench_bzip2.py 100 >> gpurun_out/rsort_ab.log 2>&1; echo "^cub" >> gpurun_out/rsort_ab.log
  timeout 300 python tools/bench_bzip2.py 100 >> gpurun_out/rsort_ab.log 2>&1; echo "^rsort" >> gpurun_out/rsort_ab.log
done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/rsort_launches.csv python tools/bench_bzip2.py 8 > gpurun_out/rsort_ncu.log 2>&1
PCBZ_LIB=paper_2310_09467_b200/_native/variants/libpcbz_cub.so timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/cub_launches.csv python tools/bench_bzip2.py 8 > gpurun_out/cub_ncu.log 2>&1
