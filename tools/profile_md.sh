#!/bin/bash
# profiles/<name>.md from an ncu --set full capture: summary table, stall
# reasons, pipe utilisation (tools/ncu_summary.py) and the opcode mix
# (tools/ncu_opmix.py).   usage: tools/profile_md.sh REP OUT.md "title"
rep=$1; out=$2; title=$3
{
  echo "# $title"
  echo
  echo "Source capture: \`$(basename $rep)\` (ncu --set full --clock-control none --import-source on, one launch)."
  echo
  python "$(dirname "$0")/ncu_summary.py" report "$rep" | tail -n +2
  echo
  echo "## Opcode mix (executed warp-instructions)"
  echo
  python "$(dirname "$0")/ncu_opmix.py" "$rep" 20
} > "$out"
