#!/bin/bash
# The reference's OWN tests (volume / mask / slicemap / render / pipeline / acceptance) on the GPU with the
# hot path rebound by install().  Run HERE first (copies the tests next to the installed reference: git-ignored,
# delete baseline/_ref_tests again afterwards), then under gpurun:  bash tools/r2_ref_suite.sh [-v] test_volume.py ...
set -u
if [ -d /root/reference/pkg/tests ]; then
  rm -rf baseline/_ref_tests && mkdir -p baseline && cp -r /root/reference/pkg/tests baseline/_ref_tests
fi
[ -d baseline/_ref_tests ] || { echo "no reference tests"; exit 1; }
python - <<'P' || exit 0
import torch, sys
sys.exit(0 if torch.cuda.is_available() else 1)
P
cd baseline/_ref_tests
NUMBA_CACHE_DIR=/tmp/ctp_ref_numba_cache PYTHONPATH=$GRAFT_REPO_ROOT/tools:$GRAFT_REPO_ROOT:$GRAFT_REPO_ROOT/baseline/_ref \
  python -m pytest "$@" -p ref_suite_plugin -p no:cacheprovider 2>&1 | tail -${CTP_REF_SUITE_TAIL:-60}
