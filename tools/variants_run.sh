python tools/stage_times.py --tag base 2>&1 | tail -1
for v in pb4 pb5 pre4 sc3 sc4 rb12 rb16 rf12; do GES_LIB=paper_2402_10128_b200/build/variants/$v/libges.so python tools/stage_times.py --tag $v 2>&1 | tail -1; done
