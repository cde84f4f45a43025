#!/bin/bash
# compute-sanitizer passes over the smoke run (every recovery kernel of both
# precisions and modalities: embed_tc, attn (dense, pruned, x3, fix-up),
# token_tc / token_x3, last_tc, combine, masklist) and a few small lossmask /
# decode / RS / baseline tests.  Summaries -> gpurun_out/sanitize_<tool>.txt
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
TESTS="tests/test_gpu_lossmask.py::test_wire_bits_are_packbits
tests/test_gpu_lossmask.py::test_undecodable_headers_raise
tests/test_gpu_codec.py::test_pframe_in_place_decode_into_reference_slot
tests/test_gpu_codec.py::test_iframe_rs_and_decode
tests/test_gpu_codec.py::test_direct_cases_match_reference
tests/test_gpu_baseline.py::test_gpu_baseline_fallback_rules"
for tool in ${TOOLS:-memcheck racecheck synccheck initcheck}; do
  out=gpurun_out/sanitize_$tool.txt
  echo "== $tool smoke" > $out
  timeout 900 compute-sanitizer --tool $tool --print-limit 20 python -c \
    "import __graft_entry__ as g; g.smoke()" >> $out 2>&1
  echo "rc=$?" >> $out
  echo "== $tool small codec / lossmask / baseline tests" >> $out
  timeout 900 compute-sanitizer --tool $tool --print-limit 20 python -m pytest -q -x $TESTS >> $out 2>&1
  echo "rc=$?" >> $out
done
