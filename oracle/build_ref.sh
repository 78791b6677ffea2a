#!/usr/bin/env bash
# Compile the REFERENCE so3 headers, where they lie under /root/reference,
# into oracle/_ref/libesref.so through the Eigen shim (oracle/ref_shim).
# Test infrastructure only; outputs only into oracle/_ref/ (git-ignored).
# No reference source is copied into this repo.
set -euo pipefail
HERE="$(cd "$(dirname "$0")" && pwd)"
REF="${EQUISTREAM_REFERENCE:-/root/reference}"
if [ ! -d "$REF/proj/include/equistream" ]; then
  echo "build_ref: $REF not present; skipping (prebuilt oracle/_ref is used if shipped)" >&2
  exit 0
fi
mkdir -p "$HERE/_ref"
g++ -std=c++20 -O2 -fPIC -shared -w \
  -I "$HERE/ref_shim/include" -I "$REF/proj/include" -I "$REF/proj/tests/support" \
  "$HERE/ref_shim/ref_wrap.cpp" -o "$HERE/_ref/libesref.so"
echo "build_ref: built $HERE/_ref/libesref.so"
