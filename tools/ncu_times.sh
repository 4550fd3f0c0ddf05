#!/bin/bash
# Per-launch device time of every scan2d* kernel of a command (ncu, cold cache,
# serialised -- compare shares, not absolutes).
# usage: tools/ncu_times.sh <skip> <count> <cmd...>
skip=$1; count=$2; shift 2
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:scan2d -s "$skip" -c "$count" --csv "$@" 2>/dev/null \
  | python3 -c '
import csv, sys
rows = [r for r in csv.reader(sys.stdin) if len(r) > 10 and r[0].isdigit()]
for r in rows:
    name = r[4].split("(")[0].replace("void ", "")
    print(f"{name:60s} {r[-2]:>6s} {r[-1]}")
'
