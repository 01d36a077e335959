#!/bin/bash
# compute-sanitizer memcheck / racecheck / synccheck over the small golden GPU
# tests (run under gpurun; logs in gpurun_out/san/, summaries copied to
# profiles/<round>/sanitizer_*.log).  bash scripts/sanitize.sh [tools...]
set -u
O=gpurun_out/san
mkdir -p $O
python -c "import sys; sys.path.insert(0,'.'); from paper_1610_07328_b200 import _native; _native.lib()"
SEL="golden or near_zero or adversarial or tie or edge_shapes or probe_candidates or summaries_codes or merge_topk or wide_band"
for tool in "${@:-memcheck racecheck synccheck}"; do
  k="$SEL"
  [ "$tool" != memcheck ] && k="test_query_golden or test_sketch_bits_golden or test_build_index_golden or merge_topk or wide_band"
  timeout 2400 compute-sanitizer --tool $tool --target-processes all --print-limit 50 --log-file $O/$tool.log \
    python -m pytest tests/test_gpu_parity.py tests/test_gpu_api.py -q -x -p no:cacheprovider -k "$k" > $O/$tool.pytest.log 2>&1
  echo "$tool rc=$? $(tail -1 $O/$tool.pytest.log)"
  grep -E "ERROR SUMMARY|RACECHECK SUMMARY|errors|hazard" $O/$tool.log | tail -3
done
