O=gpurun_out/e12; mkdir -p $O
for i in 1 2; do timeout 600 python tools/c5_f32_probe.py 300 >> $O/probeA.log 2>&1; done; cat $O/probeA.log
cp paper_2405_19246_b200/libmmot.so /tmp/libmmot_A.so; cp paper_2405_19246_b200/libmmot_B.so paper_2405_19246_b200/libmmot.so
for i in 1 2; do timeout 600 python tools/c5_f32_probe.py 300 >> $O/probeB.log 2>&1; done; cat $O/probeB.log
cp /tmp/libmmot_A.so paper_2405_19246_b200/libmmot.so
for i in 1 2; do timeout 600 python tools/c5_f32_probe.py 300 >> $O/probeA2.log 2>&1; done; cat $O/probeA2.log
MMOT_PAIR_F64=1 timeout 600 python tools/c5_f32_probe.py 300 >> $O/probeF64.log 2>&1; cat $O/probeF64.log
