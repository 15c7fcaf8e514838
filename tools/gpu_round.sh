#!/bin/bash
# One GPU-box pass: parity suite, bench (C and D), launch list, ncu --set full of the hot kernels.
# Usage (from the repo root, via gpurun): bash tools/gpu_round.sh TAG
TAG=${1:-r01}
O=gpurun_out
mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $O/${TAG}_smi.txt 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > $O/${TAG}_pytest.log 2>&1; echo "pytest rc=$?" >> $O/${TAG}_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/${TAG}_smoke.log 2>&1
timeout 600 python bench.py > $O/${TAG}_bench_C.json 2> $O/${TAG}_bench_C.err
timeout 600 python bench.py --precond D --no-cpu-baseline > $O/${TAG}_bench_D.json 2> $O/${TAG}_bench_D.err
if [ "${SKIP_NCU:-0}" != "1" ]; then
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/${TAG}_launches_C.csv \
   python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-config5 > $O/${TAG}_ncu_launch.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'k_band_lu_(res|df)' -s 0 -c 1 \
   -o $O/${TAG}_lu python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-config5 > $O/${TAG}_ncu_lu.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'k_band_lu_(res|df)' -s 0 -c 1 \
   -o $O/${TAG}_luD python bench.py --precond D --steps 1 --warmup 1 --no-cpu-baseline --no-config5 > $O/${TAG}_ncu_luD.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'k_sweep' -s 0 -c 1 \
   -o $O/${TAG}_sweep python bench.py --precond D --steps 1 --warmup 1 --no-cpu-baseline --no-config5 > $O/${TAG}_ncu_sweep.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'k_band_spmv' -s 2 -c 1 \
   -o $O/${TAG}_spmv python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-config5 > $O/${TAG}_ncu_spmv.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'k_band_spmv2' -s 0 -c 1 \
   -o $O/${TAG}_spmv2 python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-config5 > $O/${TAG}_ncu_spmv2.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file $O/${TAG}_launches_D.csv \
   python bench.py --precond D --steps 1 --warmup 1 --no-cpu-baseline --no-config5 > $O/${TAG}_ncu_launch_D.log 2>&1
fi
echo done
