# emission-kernel run-length A/B: per-launch times of the emit kernel on 100
# C2 frames (tools/profile_emit.py) for each variant built by
# tools/build_variants.py base emit_run2 emit_run8 emit_run16
rm -f gpurun_out/ab_emit.txt
for v in ${EMIT_VARIANTS:-base emit_run2 emit_run8 emit_run16 base}; do
  PCBZ_LIB=paper_2310_09467_b200/_native/variants/$v/libpcbz_b200.so timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:emit --csv python tools/profile_emit.py > gpurun_out/ab_emit_$v.csv 2>/dev/null
  echo "$v $(grep -c emit gpurun_out/ab_emit_$v.csv)" >> gpurun_out/ab_emit.txt
done
