for r in 1 2; do for v in base incptr defer incptr_defer inline incptr_inline; do
PCBZ_LIB=paper_2310_09467_b200/_native/variants/$v/libpcbz_b200.so python tools/ab_judge.py 100 2>&1 | tail -1
done; done
