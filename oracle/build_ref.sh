#!/usr/bin/env bash
# Recipe for oracle/_ref: the UNMODIFIED reference package (macrohdg, pure
# Python/numpy/scipy) installed from /root/reference/pkg into oracle/_ref.
# Test infrastructure only: bench.py's --impl reference arm and cpu_baseline
# time it on the host cores; nothing in the product imports it.
# oracle/_ref is git-ignored (no reference source in history) but not
# gpurun-ignored, so the installed copy travels to the GPU box.
set -euo pipefail
HERE="$(cd "$(dirname "$0")" && pwd)"
SRC="${1:-/root/reference/pkg}"
[ -d "$SRC" ] || { echo "build_ref.sh: $SRC absent (GPU box uses the prebuilt oracle/_ref)"; exit 0; }
TMP="$(mktemp -d)"
trap 'rm -rf "$TMP"' EXIT
# /root/reference is read-only and setuptools writes build/ + egg-info beside
# the sources: install from a scratch copy
cp -r "$SRC" "$TMP/pkg"
rm -rf "$HERE/_ref"
python -m pip install --quiet --no-index --no-build-isolation --no-deps \
    --find-links /opt/wheelhouse --target "$HERE/_ref" "$TMP/pkg"
python - "$HERE/_ref" <<'EOF'
import sys
sys.path.insert(0, sys.argv[1])
import macrohdg, macrohdg.assembly, macrohdg.solver  # noqa: F401
print("oracle/_ref: macrohdg", macrohdg.__version__, "from", macrohdg.__file__)
EOF
