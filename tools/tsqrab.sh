# A/B the load path (centre + TSQR + rank check) via tools/host_probe.py, then the GPU tests on the built lib
cp paper_1901_07643_b200/libbnreg.so /tmp/libbnreg_built.so
for f in tmpvar/lib*.so; do cp $f paper_1901_07643_b200/libbnreg.so; echo $f; for c in 4 5; do timeout 120 python tools/host_probe.py $c; done; done
cp /tmp/libbnreg_built.so paper_1901_07643_b200/libbnreg.so
timeout 900 python -m pytest -q -x tests -m gpu 2>&1 | tail -3
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"tsqr|centre" -c 4 --csv python tools/host_probe.py 4 > gpurun_out/tsqr4.csv 2>/dev/null
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"tsqr|centre" -c 4 --csv python tools/host_probe.py 5 > gpurun_out/tsqr5.csv 2>/dev/null
