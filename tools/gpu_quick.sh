#!/bin/bash
# Quick GPU-box pass: build check, parity suite (optionally filtered), one bench line.
# Usage: bash tools/gpu_quick.sh TAG [pytest -k expr]
TAG=${1:-q}
O=gpurun_out
mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $O/${TAG}_smi.txt 2>&1
if [ -n "$2" ]; then K=(-k "$2"); else K=(); fi
timeout 1500 python -m pytest tests -m gpu -x -q "${K[@]}" > $O/${TAG}_pytest.log 2>&1; echo "pytest rc=$?" >> $O/${TAG}_pytest.log
timeout 600 python bench.py --no-cpu-baseline > $O/${TAG}_bench_C.json 2> $O/${TAG}_bench_C.err
echo done
