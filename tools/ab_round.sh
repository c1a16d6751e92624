# A/B of library variants (tools/build_variants.py) on 100 C2 frames, 2 rounds
for r in 1 2; do for v in ${VARIANTS:-base}; do
PCBZ_LIB=paper_2310_09467_b200/_native/variants/$v/libpcbz_b200.so python tools/ab_judge.py 100 2>&1 | tail -1
done; done
