#!/bin/bash
# Runs on a GPU box (via gpurun): tests, bench (both arms), the ncu launch list of a short bench and
# `ncu --set full` captures of the dominant kernels (decode, ingest, drift-regime maintenance).
# Outputs land in gpurun_out/<tag>/ (scratch); scripts/summarize_profiles.py <tag> writes the
# summaries into profiles/.
set -u
OUT=gpurun_out/${1:-r2}
mkdir -p "$OUT"
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,clocks.mem --format=csv > "$OUT/gpu.txt" 2>&1
lscpu | grep -E "Model name|^CPU\(s\)" > "$OUT/cpu.txt" 2>&1
timeout 1500 python -m pytest tests -m gpu -q > "$OUT/pytest_gpu.txt" 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > "$OUT/smoke.txt" 2>&1
timeout 900 python bench.py > "$OUT/bench.json" 2> "$OUT/bench.err"
timeout 900 python bench.py --impl reference > "$OUT/bench_reference.json" 2> "$OUT/bench_reference.err"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none \
  -k regex:"k_(attend|score_select|select3|resolve|approx|topm|assign|build_cands|store_rows|ring_write|append|tier|tok|split)" -c 800 --csv \
  --log-file "$OUT/launches.csv" python bench.py --steps 5 --warmup 3 --frames 5 --no-cpu-baseline --no-offload --no-streams --no-config4 > "$OUT/ncu_launch.log" 2>&1
# decode kernels (skip the warm-up launches), then ingest kernels (absorb regime), then the
# drift regime's maintenance kernels (relaunch resolve + split k-means)
timeout 1200 ncu --set full --clock-control none --import-source on \
  -k regex:"k_(attend|select3|score_select)" -s 6 -c 2 -o "$OUT/full_decode" \
  python bench.py --steps 5 --warmup 3 --frames 5 --no-cpu-baseline --no-offload --no-streams --no-config4 > "$OUT/ncu_full_decode.log" 2>&1
timeout 1200 ncu --set full --clock-control none --import-source on \
  -k regex:"k_(resolve_spec|assign_tc)" -s 12 -c 2 -o "$OUT/full_ingest" \
  python bench.py --steps 5 --warmup 3 --frames 5 --no-cpu-baseline --no-offload --no-streams --no-config4 > "$OUT/ncu_full_ingest.log" 2>&1
timeout 1200 ncu --set full --clock-control none --import-source on \
  -k regex:"k_(resolve|split_two_batch)$" -s 30 -c 3 -o "$OUT/full_drift" \
  python scripts/drift_profile.py 16 8 > "$OUT/ncu_full_drift.log" 2>&1
DRIFT_TIMING=1 timeout 600 python scripts/drift_profile.py 112 12 > "$OUT/drift_profile.json" 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_tok_(approx|select|gather)|k_attend" -c 40 --csv \
  --log-file "$OUT/launches_token.csv" python scripts/kernel_times.py token 3 > "$OUT/ncu_launch_token.log" 2>&1
timeout 600 python scripts/split_time.py > "$OUT/split_time.txt" 2>&1
KVC_BUILD_TIMING=1 timeout 900 python scripts/build_time.py 112 32 > "$OUT/build_time.txt" 2>&1
ls -la "$OUT"
