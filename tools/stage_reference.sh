#!/usr/bin/env bash
# Stage the unmodified reference next to the repo, git-ignored (baseline/_ref):
# the pip-installed package (bench.py --impl reference) and a copy of its test
# suite (tests/test_gpu_reference_suite.py). Run in the build container, where
# /root/reference exists; gpurun ships baseline/_ref to the GPU box.
set -euo pipefail
ROOT="$(cd "$(dirname "$0")/.." && pwd)"
TMP="$(mktemp -d)"
cp -r /root/reference/pkg "$TMP/pkg"
python -m pip install --no-index --no-build-isolation --no-deps --find-links /opt/wheelhouse \
  --target "$ROOT/baseline/_ref" "$TMP/pkg" >/dev/null
mkdir -p "$ROOT/baseline/_ref/reference_tests"
cp /root/reference/pkg/tests/*.py "$ROOT/baseline/_ref/reference_tests/"
rm -rf "$TMP"
echo "staged: $(ls "$ROOT/baseline/_ref")"
