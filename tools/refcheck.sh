#!/bin/bash
# Run the REFERENCE's own test suite (pkg/tests, unmodified) against this
# drop-in through a `b2sr` import shim -- verification only.
#
#   bash tools/refcheck.sh prepare      (build container: /root/reference exists)
#   bash tools/refcheck.sh run          (GPU box: the snapshot carries .refcheck/)
#
# `prepare` stages the reference's tests and its numpy test oracle
# (b2sr/reference.py, which the tests import) into .refcheck/ -- a scratch
# directory listed in .gitignore, never committed -- next to a shim package
# whose `b2sr` modules ARE paper_2201_08560_b200's.  The results are what
# gets committed (profiles/r02_refcheck.txt).
set -euo pipefail
ROOT=$(cd "$(dirname "$0")/.." && pwd)
D="$ROOT/.refcheck"
case "${1:-run}" in
prepare)
    R=/root/reference/pkg
    rm -rf "$D"
    mkdir -p "$D/shim/b2sr"
    cp -r "$R/tests" "$D/tests"
    cp "$R/src/b2sr/reference.py" "$D/shim/b2sr/reference.py"
    cat > "$D/shim/b2sr/__init__.py" <<'PY'
"""`import b2sr` -> the B200 drop-in (paper_2201_08560_b200)."""
import importlib
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[3]))
from paper_2201_08560_b200 import *  # noqa: F401,F403,E402
from paper_2201_08560_b200 import __all__  # noqa: E402,F401

for _m in ("formats", "kernels", "algorithms", "semirings", "cli", "matrixio", "profile", "errors"):
    sys.modules[f"{__name__}.{_m}"] = importlib.import_module(f"paper_2201_08560_b200.{_m}")
PY
    echo "staged $(ls "$D/tests" | wc -l) files in $D"
    ;;
run)
    cd "$D"
    PYTHONPATH="$D/shim" python -m pytest tests -q -p no:cacheprovider -o addopts="" "${@:2}"
    ;;
esac
