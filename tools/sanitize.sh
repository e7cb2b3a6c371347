#!/bin/bash
# compute-sanitizer passes over the small-fixture parity tests ("compute-sanitizer
# (memcheck/racecheck) on the small configs").  Run on the GPU box:
#     bash tools/sanitize.sh [outdir] [tools...]
# Each tool runs the selected tests once; its report goes to <outdir>/<tool>.log and one line per tool to
# <outdir>/summary.txt.  The multi-million-point tests are deselected (the sanitizer slows kernels 10-100x).
set -u
OUT=${1:-gpurun_out/sanitizer}
shift || true
TOOLS=${*:-memcheck racecheck synccheck}
mkdir -p "$OUT"
: > "$OUT/summary.txt"
SEL="tests/test_gpu_parity.py tests/test_csv.py"
DESEL="not adversarial and not multi_chunk and not lifecycle and not concurrent and not random_decimal"
for tool in $TOOLS; do
  t0=$(date +%s)
  timeout ${SANITIZE_TIMEOUT:-1500} compute-sanitizer --tool "$tool" --error-exitcode 99 --log-file "$OUT/$tool.log" \
    python -m pytest $SEL -m gpu -q -p no:cacheprovider -k "$DESEL" > "$OUT/$tool.pytest.log" 2>&1
  rc=$?
  t1=$(date +%s)
  {
    echo "== $tool: exit $rc, $((t1 - t0)) s"
    tail -1 "$OUT/$tool.pytest.log"
    grep -E "ERROR SUMMARY|RACECHECK SUMMARY" "$OUT/$tool.log" | tail -2
  } | tee -a "$OUT/summary.txt"
done
