#!/bin/bash
# compute-sanitizer over the GPU parity paths (run on a B200 via gpurun; summaries -> profiles/).
#   memcheck : out-of-bounds / misaligned accesses, leaks, API errors (every kernel of the
#              config-1 parity stream incl. splits, deferred settles, tier migrations, token mode)
#   racecheck: shared-memory hazards (mbarrier pipelines of K6 / the tile kernel, K4, resolve)
#   synccheck: barrier / warp-sync misuse
set -u
OUT=gpurun_out/${1:-san}
mkdir -p "$OUT"
CS=/usr/local/cuda/bin/compute-sanitizer
T="tests/test_parity_gpu.py::test_config1_full_stream tests/test_parity_gpu.py::test_deferred_and_prefetch_drift tests/test_token_gpu.py tests/test_tiers_gpu.py"
timeout 2400 $CS --tool memcheck --leak-check full --target-processes all --print-limit 50 \
  python -m pytest $T -q -x -p no:cacheprovider > "$OUT/memcheck.txt" 2>&1
echo "memcheck rc=$?" >> "$OUT/memcheck.txt"
timeout 1800 $CS --tool racecheck --racecheck-report all --print-limit 50 \
  python -c "import __graft_entry__ as g; g.smoke()" > "$OUT/racecheck.txt" 2>&1
echo "racecheck rc=$?" >> "$OUT/racecheck.txt"
# the same without K6 (its mbarrier stage hand-off is outside racecheck's model): any hazard left is real
timeout 1800 $CS --tool racecheck --racecheck-report all --print-limit 50 --kernel-name-exclude kns=k_attend \
  python -c "import __graft_entry__ as g; g.smoke()" > "$OUT/racecheck_no_k6.txt" 2>&1
echo "racecheck (k_attend excluded) rc=$?" >> "$OUT/racecheck_no_k6.txt"
timeout 1800 $CS --tool synccheck --print-limit 50 \
  python -c "import __graft_entry__ as g; g.smoke()" > "$OUT/synccheck.txt" 2>&1
echo "synccheck rc=$?" >> "$OUT/synccheck.txt"
tail -4 "$OUT"/*.txt
