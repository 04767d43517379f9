#!/bin/bash
# Shard timing and standalone complex-sweep launch durations for the
# diagonal-sweep variants at the 1/8 and 1/4 shards (diagnostics).
for cfg in "32,16,32,16:0" "32,16,32,16:8" "32,16,16,16:0" "32,16,16,16:8" "32,16,16,16:4"; do
  d=${cfg%%:*}; rx=${cfg##*:}
  echo "== HSRQ_DIAG=$d HSRQ_DIAG_RX=$rx"
  HSRQ_DIAG=$d HSRQ_DIAG_RX=$rx timeout 300 python tools/shard_time.py 4 8
  HSRQ_DIAG=$d HSRQ_DIAG_RX=$rx timeout 300 /usr/local/cuda/bin/ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k_diag_cplx -s 100 -c 6 --csv python tools/shard_time.py 8 2>/dev/null | grep k_diag | awk -F'","' '{print $5, $NF}' | tail -3
done
