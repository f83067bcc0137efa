#!/bin/bash
# One validation pass on a 1-GPU box (dev tool): GPU suite, bench (our arm +
# reference arm), then -- only after the plain runs exited 0 -- the ncu
# launch list of the bench command and one ncu --set full capture of the
# GEMVs at the full Cascadia shape.  Outputs under gpurun_out/$TAG.
TAG=${1:-r02}
O=gpurun_out/$TAG
mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv > $O/smi.txt
timeout 1500 python -m pytest tests -m gpu -q -rfEs --durations=25 > $O/tests.log 2>&1; echo "tests rc=$?" >> $O/tests.log
timeout 900 python bench.py > $O/bench.json 2> $O/bench.err; brc=$?; echo "bench rc=$brc"
timeout 900 python bench.py --impl reference > $O/ref.json 2> $O/ref.err; echo "ref rc=$?"
if [ $brc -eq 0 ]; then
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv \
      --log-file $O/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-parity \
      > $O/ncu_launch.log 2>&1; echo "ncu launches rc=$?"
  timeout 1200 ncu --set full --clock-control none --import-source on -k regex:gemv -s 2 -c 2 \
      -o $O/gemv_full python tools/profile_gemv.py 32768 > $O/ncu_gemv.log 2>&1; echo "ncu gemv rc=$?"
fi
tail -3 $O/tests.log
