#!/bin/bash
# Standard GPU round-trip: build, kernel+model tests, short bench, launch list.
python -m paper_2306_06446_b200.build > gpurun_out/build.log 2>&1 || { tail gpurun_out/build.log; exit 1; }
timeout 600 python -m pytest tests -m gpu -q -x --timeout 300 -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1
tail -4 gpurun_out/pytest_gpu.log
timeout 400 python bench.py --steps 10 --warmup 3 --skip-cpu > gpurun_out/bench.log 2>&1
head -c 330 gpurun_out/bench.log; echo
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv --log-file gpurun_out/launches.csv python scripts/profile_forward.py > gpurun_out/ncu1.log 2>&1
