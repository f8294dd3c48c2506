#!/bin/bash
# A/B of an environment switch on the AGNN layer (tools/agnn_only.py):
#   bash tools/ab_env.sh "VAR=value" [agnn_only args]
# prints default / switched timings, twice, plus the dense-only / sparse-only parts.
sw=$1; shift
for r in 1 2; do
  for which in default switched; do
    if [ $which = default ]; then e=""; else e="$sw"; fi
    echo "$which: $(env $e python tools/agnn_only.py "$@" 2>&1 | tail -1)"
  done
done
for m in 1 2; do
  for which in default switched; do
    if [ $which = default ]; then e=""; else e="$sw"; fi
    echo "dbg$m $which: $(env $e SGTK_PANEL_DEBUG=$m python tools/agnn_only.py "$@" 2>&1 | tail -1)"
  done
done
