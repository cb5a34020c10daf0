#!/usr/bin/env bash
# Re-measure every number quoted in profiles/r1_results.md / r2_results.md on one B200, into
# gpurun_out/refresh/ (copy what you want to keep into profiles/).  Run through
#   gpurun --timeout 2400 -- 'bash tools/refresh_profiles.sh'
# Each step is bounded by its own timeout so one failure does not stall the rest.
set -u
OUT=gpurun_out/refresh
mkdir -p "$OUT"
run() {  # name, timeout, command...
  local name=$1 t=$2
  shift 2
  echo "== $name" >&2
  timeout "$t" "$@" > "$OUT/$name.log" 2>&1 || echo "$name failed (rc=$?)" >&2
}
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw,temperature.gpu --format=csv > "$OUT/gpu.csv"
run bench 600 python bench.py
run bench_reference 600 python bench.py --impl reference
for w in 13b-8k 70b-16k; do run "bench_$w" 600 python bench.py --workload "$w" --no-cpu-baseline --no-extras; done
run migrate_vs_library 600 python tools/bench_migrate_baselines.py
run host_link 300 python tools/bench_host_link.py
run interference 300 python tools/bench_interference.py
run copy_sms_bulk 300 python tools/bench_copy_sms.py
run copy_sms_ldg 300 python tools/bench_copy_sms.py --engine ldg
run launch_gap 300 python tools/bench_launch_gap.py
run reprefill_rounds 300 python tools/bench_reprefill_rounds.py
run concurrent 600 python tools/bench_concurrent.py
for a in "" "--rows 4096" "--shape llama2-7b --rows 2048" "--kv-only" "--rows 1456" "--rows 1280"; do
  run "reprefill_${a// /_}" 300 python tools/bench_reprefill.py $a
done
run split 600 python tools/bench_split.py
run issue 600 python tools/bench_issue.py
run foreign 600 python tools/bench_foreign.py
run pipelined_decode 600 python tools/bench_pipelined_decode.py
run split_power 600 python tools/probe_split_power.py
run live 600 python tools/bench_live.py
for a in "" "--layers 1" "--shape llama3-70b-gqa --seq 16384" "--shape llama3-70b-gqa --seq 16384 --layers 1" \
         "--shape llama2-13b --seq 8192" "--batch 8 --layers 4"; do
  run "decode_${a// /_}" 120 python tools/bench_decode.py $a
done
run decode_vs_flashinfer 900 python tools/bench_decode_vs_flashinfer.py
run scheduler 900 python tools/bench_scheduler.py --seeds 0 1 2
run online_loop 900 python tools/online_loop.py
echo "done: $(ls "$OUT" | wc -l) files in $OUT" >&2
