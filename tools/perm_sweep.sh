#!/bin/bash
# Sweep the permute tile run thresholds (TNX_PERM_SRC / TNX_PERM_DST) on the two
# perm microbenchmarks; per-launch kernel times from an ncu launch list.
CFGS=("32 32")
[ -n "$PERM_CFGS" ] && IFS=, read -ra CFGS <<< "$PERM_CFGS"
for cfg in "${CFGS[@]}"; do
  set -- $cfg
  for script in tools/run_perm.py tools/run_perm_hoist.py; do
    TNX_PERM_SRC=$1 TNX_PERM_DST=$2 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
      --clock-control none -k regex:"perm|pack_kernel" --csv python $script 1 2>/dev/null \
      | grep -E "gpu__time|dram__bytes" | awk -F'","' -v c="$1/$2" -v s=$(basename $script) '{print c, s, $5, $(NF-2), $NF}'
  done
done
