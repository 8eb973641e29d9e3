#!/bin/bash
# Dev validation (not part of the driver's tests): run the reference package's
# own pytest suite against the B200 drop-in through an `lsopc` shim.
#   prep  (build container, where /root/reference exists): copies the reference
#         tests into the git-ignored baseline/_ref/ (never committed)
#   run   (GPU box): pytest with the shim first on PYTHONPATH
set -e
ROOT=$(cd "$(dirname "$0")/.." && pwd)
REF=$ROOT/baseline/_ref
case "$1" in
  prep)
    rm -rf "$REF/tests" "$REF/shim"
    mkdir -p "$REF/shim/lsopc"
    cp -r /root/reference/pkg/tests "$REF/tests"
    cat > "$REF/shim/lsopc/__init__.py" <<'PY'
# shim: `import lsopc` -> the B200 drop-in, every module including cli / fileio
import sys
import paper_2303_12529_b200 as _b2
from paper_2303_12529_b200 import *  # noqa
from paper_2303_12529_b200 import cli, errors, fields, fileio, levelset, litho, metrics, optimizer  # noqa
for _m in ("cli", "errors", "fields", "fileio", "levelset", "litho", "metrics", "optimizer"):
    sys.modules["lsopc." + _m] = getattr(_b2, _m)
PY
    echo "prepared $REF" ;;
  run)
    cd "$REF"
    PYTHONPATH="$REF/shim:$ROOT" LSOPC_B200_PRECISION=${PREC:-fp64} NUMBA_CACHE_DIR=/tmp/numba \
      python -m pytest tests -q -p no:cacheprovider ${PYTEST_ARGS} ;;
  *) echo "usage: $0 prep|run"; exit 2 ;;
esac
