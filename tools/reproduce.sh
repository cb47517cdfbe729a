#!/usr/bin/env bash
# Regenerate the measurements DESIGN.md quotes, on one B200 (run from the repo root,
# e.g. through gpurun).  Outputs land in gpurun_out/<mode>/; copy what you want judged
# into profiles/.  Modes (default: all):
#   all       every bench line, suite and tool DESIGN.md cites, + kernel evidence
#   evidence  the headline bench lines + the ncu launch list and the full capture of
#             the dominant kernel (what a kernel change needs re-measured)
#   tests     pytest -m gpu, smoke, the reference's own suite (three bindings)
#   parts     part isolation of the fused recompute: probe builds (tools/probe_builds.py)
#             with FS_RC_* macros that drop one part each (timings of probe builds are
#             NOT results); the shipped library is not touched
#   sanitize  compute-sanitizer memcheck / racecheck / synccheck over every kernel family
set -euo pipefail
MODE=${1:-all}
O=gpurun_out/$MODE
mkdir -p "$O"
python -c "import __graft_entry__ as g; g.build()"

tests() {
  python -c "import __graft_entry__ as g; g.smoke()"                        > "$O/smoke.log"
  python -m pytest tests -q -m gpu                                          > "$O/pytest_gpu.log" || true
  python tools/run_reference_tests.py                                       > "$O/reference_suite.log" 2>&1 || true
  python tools/run_reference_tests.py --boundary-only                       > "$O/reference_suite_boundary.log" 2>&1 || true
  python tools/run_reference_tests.py --bind-streaming                      > "$O/reference_suite_streaming.log" 2>&1 || true
}

evidence() {
  python bench.py                                                           > "$O/bench_c2.json"
  python bench.py --impl reference                                          > "$O/bench_c2_reference.json"
  python bench.py --config c3 --no-cpu                                      > "$O/bench_c3.json"
  # kernel evidence: the launch list of the bench command and one full capture of the
  # dominant kernel (numbers printed under ncu are not bench values)
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
      --log-file "$O/launches_c2.csv" \
      python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu                > /dev/null
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_recompute_f4 -s 2 -c 1 \
      -o "$O/c2_recompute_fused" python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu > /dev/null
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_pack_flat -s 8 -c 1 \
      -o "$O/c2_pack_flat" python bench.py --steps 1 --warmup 3 --no-cpu > /dev/null
}

parts() {
  local cases=256:8192:8192,129:8192:8192
  python tools/probe_builds.py nomma="-DFS_RC_NO_MMA" nocount="-DFS_RC_NO_COUNT" \
      noexp="-DFS_RC_NO_EXPAND" noemit="-DFS_RC_NO_EMIT" noload="-DFS_RC_NO_LOAD" \
      nopf="-DFS_RC_L2PF=0" batch1="-DFS_RC_BATCH=1" > /dev/null
  for v in base nomma nocount noexp noemit noload nopf batch1; do
    echo "# $v" >> "$O/parts.jsonl"
    if [ "$v" = base ]; then
      python tools/k_sweep.py --fused-only --cases $cases >> "$O/parts.jsonl" 2>&1
    else
      FS_LIB_PROBE="probes/$v.so" python tools/k_sweep.py --fused-only --cases $cases >> "$O/parts.jsonl" 2>&1
    fi
  done
}

sanitize() {
  for tool in memcheck racecheck synccheck; do
    compute-sanitizer --tool "$tool" python tools/sanitize_cases.py         > "$O/$tool.log" 2>&1 || true
  done
}

case "$MODE" in
  tests) tests ;;
  evidence) evidence ;;
  parts) parts ;;
  sanitize) sanitize ;;
  all)
    tests
    evidence
    python bench.py --config c1                                             > "$O/bench_c1.json"
    python bench.py --config c4 --steps 3 --warmup 3                        > "$O/bench_c4.json"
    python tools/sweep_bench.py                                             > "$O/sweep_c5.json"
    python tools/dual_bench.py                                              > "$O/dual_buffer_suite.json"
    python tools/k_sweep.py                                                 > "$O/k_sweep.jsonl"
    python tools/service_bench.py                                           > "$O/service_c2.json"
    python tools/ingest_bench.py                                            > "$O/ingest.json"
    python tools/compare_with_reference.py --width 2048 --height 1536 --k 96 > "$O/compare_with_reference.json"
    sanitize
    ;;
  *) echo "unknown mode $MODE" >&2; exit 2 ;;
esac
echo "done: $O"
