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
if [ -d "$REF" ]; then
for t in test_lora test_batch_select test_workload test_memory_model; do
  g++ -std=c++20 -O1 -I "$HERE" -I "$ROOT/include" -o "$OUT/$t" "$REF/$t.cpp" "$HERE/main.cpp" \
      -L "$PKG" -lfusim_b200 -lmlora -Wl,-rpath,"$PKG"
done
else
  echo "reference tests not present ($REF); reference suites not rebuilt" >&2
fi
# façade-only driver (no reference sources needed)
g++ -std=c++20 -O1 -I "$ROOT/include" -o "$OUT/facade_forward_io" "$HERE/facade_forward_io.cpp" \
    -L "$PKG" -lfusim_b200 -lmlora -Wl,-rpath,"$PKG"
# the B200 executor behind the fused iteration, driven by a simulator-shaped loop
g++ -std=c++20 -O1 -I "$ROOT/include" -o "$OUT/executor_loop" "$HERE/executor_loop.cpp" \
    -L "$PKG" -lfusim_b200 -lmlora -Wl,-rpath,"$PKG"
echo "built: $(ls "$OUT")"
