# A/B the best-subsets transform: time each tmpvar/lib*.so at cfg5 and cfg4, then run its tests on the built lib
cp paper_1901_07643_b200/libbnreg.so /tmp/libbnreg_built.so
for f in tmpvar/lib*.so; do cp $f paper_1901_07643_b200/libbnreg.so; for c in 5 4; do echo $f; timeout 120 python tools/bps_time.py $c; done; done
cp /tmp/libbnreg_built.so paper_1901_07643_b200/libbnreg.so
timeout 900 python -m pytest -q -x tests/test_gpu_parity.py -k best_subsets 2>&1 | tail -3
timeout 900 python -m pytest -q -x tests/test_gpu_fullsize.py -k best_subsets 2>&1 | tail -3
