#!/bin/bash
# Source-level ncu captures of the persistent batched kernel: C2 (one instance, latency-bound) and
# the C5 probe (1184 instances x 30 sweeps).  Reports + per-line source CSVs land in $OUT.
O=${OUT:-gpurun_out/src}
mkdir -p $O
if [ -n "$TESTS" ]; then timeout 900 python -m pytest $TESTS -q -x > $O/pytest.log 2>&1; echo "pytest rc=$?" >> $O/pytest.log; tail -3 $O/pytest.log; fi
CMD2="python bench.py --config C2 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e"
timeout 300 $CMD2 > $O/c2_plain.json 2>&1; echo "c2 rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_bat_sinkhorn -c 1 -o $O/prof_c2 $CMD2 > $O/ncu_c2.log 2>&1; echo "ncu c2 rc=$?"
ncu -i $O/prof_c2.ncu-rep --page source --csv > $O/src_c2.csv 2>/dev/null
if [ "${C5:-1}" = "1" ]; then
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_bat_sinkhorn -c 1 -o $O/prof_c5 python tools/c5_probe.py 1184 30 > $O/ncu_c5.log 2>&1; echo "ncu c5 rc=$?"
ncu -i $O/prof_c5.ncu-rep --page source --csv > $O/src_c5.csv 2>/dev/null
python tools/prof_summary.py $O/prof_c5.ncu-rep > $O/summary_c5.txt 2>&1
rm -f $O/prof_c5.ncu-rep
fi
python tools/prof_summary.py $O/prof_c2.ncu-rep > $O/summary_c2.txt 2>&1
ls -la $O
