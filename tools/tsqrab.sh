# A/B the load path (centre + TSQR + rank check): TSQR kernel time (ncu) and the step (host_probe), then GPU tests
cp paper_1901_07643_b200/libbnreg.so /tmp/libbnreg_built.so
for f in tmpvar/lib*.so; do cp $f paper_1901_07643_b200/libbnreg.so; echo $f; for c in 4 5; do timeout 120 python tools/host_probe.py $c 2>&1 | grep step
  timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:tsqr -c 2 --csv python tools/host_probe.py $c 2>/dev/null | grep tsqr_kernel | tail -1 | awk -F'"' '{print "tsqr ns", $(NF-1)}'; done; done
cp /tmp/libbnreg_built.so paper_1901_07643_b200/libbnreg.so
timeout 900 python -m pytest -q -x tests -m gpu 2>&1 | tail -3
