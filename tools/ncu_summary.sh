#!/bin/bash
# ncu_summary.sh REP OUT: the raw metrics of every profiled launch of REP as CSV (small enough to
# bring back from the GPU box; the .ncu-rep itself may not be).
ncu -i "$1" --page raw --csv > "$2" 2>/dev/null
