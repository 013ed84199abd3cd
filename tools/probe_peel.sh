timeout 1500 python -m pytest tests -m gpu -q -x 2>&1 | tail -3
bash tools/gpu_variant_ab2.sh "" "-DTF_PEEL_NO_EARLY_STOP"
python -m paper_2011_03910_b200._build --force > /dev/null 2>&1
