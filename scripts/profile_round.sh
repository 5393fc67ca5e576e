#!/bin/bash
# Runs on a GPU box (via gpurun): tests, bench (both arms), the ncu launch list of a short bench and
# one `ncu --set full` capture of the dominant kernels. Outputs land in gpurun_out/ (scratch);
# summaries are copied into profiles/ by scripts/summarize_profiles.py on the build host.
set -u
OUT=gpurun_out/${1:-r1}
mkdir -p "$OUT"
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,clocks.mem --format=csv > "$OUT/gpu.txt" 2>&1
timeout 900 python -m pytest tests -m gpu -q > "$OUT/pytest_gpu.txt" 2>&1
timeout 900 python bench.py > "$OUT/bench.json" 2> "$OUT/bench.err"
timeout 900 python bench.py --impl reference > "$OUT/bench_reference.json" 2> "$OUT/bench_reference.err"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none \
  -k regex:"k_(attend|score_select|select3|resolve|approx|topm|assign|build_cands|store_rows|ring_write|append|tier|tok)" -c 600 --csv \
  --log-file "$OUT/launches.csv" python bench.py --steps 5 --warmup 3 --frames 5 --no-cpu-baseline --no-offload --no-streams > "$OUT/ncu_launch.log" 2>&1
# decode kernels (skip the warm-up launches), then ingest kernels
timeout 1200 ncu --set full --clock-control none --import-source on \
  -k regex:"k_(attend|select3|score_select)" -s 6 -c 2 -o "$OUT/full_decode" \
  python bench.py --steps 5 --warmup 3 --frames 5 --no-cpu-baseline --no-offload --no-streams > "$OUT/ncu_full_decode.log" 2>&1
timeout 1200 ncu --set full --clock-control none --import-source on \
  -k regex:"k_(resolve|assign|approx|topm)" -s 12 -c 3 -o "$OUT/full_ingest" \
  python bench.py --steps 5 --warmup 3 --frames 5 --no-cpu-baseline --no-offload --no-streams > "$OUT/ncu_full_ingest.log" 2>&1
ls -la "$OUT"
# token-level baseline kernels (config-5 shape, one stream)
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_tok_(approx|select|gather)|k_attend" -c 40 --csv \
  --log-file "$OUT/launches_token.csv" python scripts/kernel_times.py token 3 > "$OUT/ncu_launch_token.log" 2>&1
# maintenance / build slow paths on the GPU: split k-means, drift ingest, batch build
timeout 600 python scripts/split_time.py > "$OUT/split_time.txt" 2>&1
timeout 900 python scripts/drift_ingest.py 0.05 10 16 > "$OUT/drift_ingest.json" 2> "$OUT/drift_ingest.err"
KVC_BUILD_TIMING=1 BUILD_HOST_TOO=1 timeout 900 python scripts/build_time.py 16 32 > "$OUT/build_time.txt" 2>&1
KVC_BUILD_TIMING=1 timeout 900 python scripts/build_time.py 112 32 >> "$OUT/build_time.txt" 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_kmeans" -c 1 -o "$OUT/full_kmeans" \
  python scripts/build_time.py 16 32 > "$OUT/ncu_full_kmeans.log" 2>&1
ls -la "$OUT"
