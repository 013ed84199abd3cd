timeout 900 python -m pytest tests/test_gpu_units.py tests/test_gpu_ties.py tests/test_gpu_tracker.py -q -x -m gpu 2>&1 | tail -3
bash tools/gpu_variant_ab2.sh "" "-DTF_CTA_LAP_NOINLINE"
