#!/usr/bin/env bash
# Builds oracle/_ref/ref_golden from the reference's own headers (inline
# definitions only -- the reference has no src/) and regenerates
# tests/golden/ref_inline.json.  Needs /root/reference (build container only).
set -euo pipefail
here="$(cd "$(dirname "$0")" && pwd)"
ref="${REFERENCE_ROOT:-/root/reference}/proj/include"
[ -d "$ref" ] || { echo "reference headers not found at $ref" >&2; exit 1; }
mkdir -p "$here/_ref"
/usr/bin/g++ -std=c++20 -O1 -ffp-contract=off -I"$ref" "$here/ref_golden.cpp" -o "$here/_ref/ref_golden"
"$here/_ref/ref_golden" > "$here/../tests/golden/ref_inline.json"
echo "wrote tests/golden/ref_inline.json"
