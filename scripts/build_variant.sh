#!/bin/bash
# build_variant.sh NAME [MACRO=VALUE ...]: build liborloj with extra -D flags into
# build_variants/liborloj_NAME.so (load it with ORLOJ_LIB=... for experiments).
set -e
ROOT=$(cd "$(dirname "$0")/.." && pwd)
NAME=$1; shift
cd "$ROOT"
python - "$NAME" "$@" <<'PY'
import sys
from paper_2209_00159_b200 import _abi
name, defs = sys.argv[1], sys.argv[2:]
print(_abi.build(out=f"build_variants/liborloj_{name}.so", defines=defs))
PY
