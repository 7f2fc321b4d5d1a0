#!/usr/bin/env bash
# Compile the reference's own unit suites (read in place from /root/reference,
# never copied) against the B200 façade headers in include/fusim/ and link them
# to the façade + C-ABI libraries.  Binaries land in tests/cpp/build/ (ignored
# by git, shipped to the GPU box by gpurun).
set -euo pipefail
HERE="$(cd "$(dirname "$0")" && pwd)"
ROOT="$(cd "$HERE/../.." && pwd)"
REF="${REF:-/root/reference/proj/tests}"
PKG="$ROOT/paper_2312_02515_b200"
OUT="$HERE/build"
mkdir -p "$OUT"
[ -d "$REF" ] || { echo "reference tests not present ($REF); using prebuilt binaries" >&2; exit 0; }
for t in test_lora test_batch_select test_workload; do
  g++ -std=c++20 -O1 -I "$HERE" -I "$ROOT/include" -o "$OUT/$t" "$REF/$t.cpp" "$HERE/main.cpp" \
      -L "$PKG" -lfusim_b200 -lmlora -Wl,-rpath,"$PKG"
done
echo "built: $(ls "$OUT")"
