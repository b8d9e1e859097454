#!/bin/bash
# Round evidence: GPU tests, smoke, every config's bench line, reference arm, C4 launch list + ncu of
# the update kernel, C5 ncu of the pair kernel (full batch, 10 sweeps), C3 launch list.
O=${OUT:-gpurun_out/final}
mkdir -p $O
if [ "${SKIP_TESTS:-0}" != "1" ]; then
timeout 2400 python -m pytest tests -m gpu -q -rf --durations=25 > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
tail -4 $O/pytest_gpu.log
fi
python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; tail -1 $O/smoke.log
timeout 600 python bench.py > $O/bench_c4.json 2> $O/bench_c4.err; echo "c4 rc=$?"
timeout 600 python bench.py --impl reference > $O/bench_c4_ref.json 2> $O/bench_c4_ref.err; echo "c4 ref rc=$?"
for c in C1 C2 C3 C3f C5; do timeout 900 python bench.py --config $c > $O/bench_$c.json 2> $O/bench_$c.err; echo "$c rc=$?"; done
timeout 600 python bench.py --config C5 --impl reference > $O/bench_c5_ref.json 2> $O/bench_c5_ref.err; echo "c5 ref rc=$?"
CMD="python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e"
timeout 300 $CMD > $O/plain.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 800 --csv --log-file $O/launches_c4.csv $CMD > $O/ncu_launch.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_sw_apply -s 20 -c 1 -o $O/prof_c4 $CMD > $O/ncu_c4.log 2>&1
CMD3="python bench.py --config C3 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file $O/launches_c3.csv $CMD3 > $O/ncu_launch3.log 2>&1
# C5: the pair family's whole-solve kernel on the full batch, 10 sweeps (the bench's 300 would replay for minutes)
timeout 300 python tools/c5_f32_probe.py 10 > $O/c5probe.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_pair_sinkhorn -c 1 -o $O/prof_c5 python tools/c5_f32_probe.py 10 > $O/ncu_c5.log 2>&1
python tools/prof_summary.py $O/launches_c4.csv $O/prof_c4.ncu-rep > $O/summary_c4.txt 2>&1
python tools/prof_summary.py $O/launches_c3.csv > $O/summary_c3.txt 2>&1
python tools/prof_summary.py $O/prof_c5.ncu-rep > $O/summary_c5.txt 2>&1
ls -la $O/*.ncu-rep 2>/dev/null
rm -f $O/prof_c5.ncu-rep $O/prof_c4.ncu-rep
echo done
