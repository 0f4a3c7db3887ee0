# NOTE: compute-sanitizer is closed on the GPU pool from round 2 on (gpurun refuses it); the last
# sanitizer evidence is profiles/r2c_sanitizer.txt.
S="compute-sanitizer --error-exitcode 9 --print-limit 20"
run(){ tool=$1; shift; echo "=== $tool $*"; timeout 900 $S --tool $tool python -m pytest -q -x "$@" 2>&1 | grep -E "passed|failed|ERROR SUMMARY|hazard|Invalid|error" | tail -6; }
run memcheck tests/test_parity_gpu.py -k "structure_block8k or rates_stage_A_and_B_S0 or dense_windows_global_mode or alg2_stale or crater_body"
CRM_LIST_ORDER=scan run memcheck tests/test_list_order_gpu.py tests/test_active_gpu.py -k "permutation or active_set"
run memcheck tests/test_parity_gpu.py -k "alg2_ps10 or crater_body"
run racecheck tests/test_parity_gpu.py -k "structure_block8k and 0.05"
run racecheck tests/test_parity_gpu.py -k "rates_stage_A_and_B_S0"
run synccheck tests/test_parity_gpu.py -k "rates_stage_A_and_B_S0 or dense_windows"
run initcheck tests/test_parity_gpu.py -k "rates_stage_A_and_B_S0 or structure_block8k"
run memcheck tests/test_multi_gpu.py -k "graph_replay or migration"
run racecheck tests/test_multi_gpu.py -k "graph_replay"
