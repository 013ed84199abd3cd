# compute-sanitizer memcheck over smoke() and a handful of parity tests (cluster association,
# narrow two-per-SM association, multi-stream, dense scene, JDE extensions). Each leg under its
# own timeout; the summaries (ERROR SUMMARY lines) are what is kept.
set -x
T=${1:-r02v}
S="compute-sanitizer --tool memcheck --print-limit 5"
timeout 500 $S python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${T}_mc_smoke.log 2>&1; echo mc_smoke=$?
timeout 900 $S python -m pytest tests/test_gpu_heads.py -q -m gpu -x -k "cfg0_single or multi_stream_cfg3_like or narrow_association_ctas_match or jde_extensions_match" > gpurun_out/${T}_mc_tests.log 2>&1; echo mc_tests=$?
grep -h "ERROR SUMMARY\|passed\|failed\|smoke ok\|Invalid\|Error:" gpurun_out/${T}_mc_*.log | head -40 > gpurun_out/${T}_memcheck.txt
cat gpurun_out/${T}_memcheck.txt
