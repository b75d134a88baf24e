#!/bin/bash
# SM clock and board power while a command runs (samples above 300 W only, i.e.
# while the GPU is busy): tools/power_probe.sh CMD...
nvidia-smi --query-gpu=clocks.sm,power.draw --format=csv,noheader,nounits -lms 100 > /tmp/pp.$$ &
S=$!
"$@"
kill $S
awk -F, '$2 > 300 {print $1, $2}' /tmp/pp.$$ | sort -n -k1 | awk '{c[NR]=$1; p[NR]=$2} END {if (NR) print "busy samples", NR, "median clock", c[int((NR+1)/2)], "MHz; power", p[int((NR+1)/2)], "W"; else print "no busy samples"}'
