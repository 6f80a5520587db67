#!/bin/bash
# Run tools/ntt_probe.py against every experimental library build in lib/variants/.
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
for so in paper_2603_22437_b200/lib/variants/*.so; do
  echo "=== $(basename "$so")"
  MMFHE_LIB="$PWD/$so" python tools/ntt_probe.py "${1:-10}" 2>&1 | tail -12
done
