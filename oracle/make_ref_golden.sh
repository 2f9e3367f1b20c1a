#!/usr/bin/env bash
# TEST INFRASTRUCTURE ONLY. Compiles oracle/ref_golden.cpp against the
# reference's Eigen-free headers (read in place under /root/reference, never
# copied) into oracle/_ref/, and regenerates tests/golden/rng_ref.json.
set -euo pipefail
here="$(cd "$(dirname "$0")" && pwd)"
ref="${VMFA_REFERENCE:-/root/reference}/proj/include"
mkdir -p "$here/_ref"
g++ -std=c++20 -O2 -I"$ref" "$here/ref_golden.cpp" -o "$here/_ref/ref_golden"
if [[ "${1:-}" == "--write" ]]; then
  "$here/_ref/ref_golden" > "$here/../tests/golden/rng_ref.json"
fi
