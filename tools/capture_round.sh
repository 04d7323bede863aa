#!/bin/bash
# The round's committed evidence in one GPU session (run under gpurun): default bench line, the
# ncu launch list of the same command, one ncu --set full capture of the chain on 200k M5
# instances.  Then, here: python tools/make_profiles.py <round> gpurun_out/cap/chain.ncu-rep
#   gpurun_out/cap/launches.csv gpurun_out/cap/bench.json
out=gpurun_out/cap
mkdir -p $out
python bench.py > $out/bench.log 2>&1
grep '^{' $out/bench.log | tail -1 > $out/bench.json
ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file $out/launches.csv \
  python bench.py --steps 2 --warmup 1 --profile-run --no-secondary > $out/launches.log 2>&1
ncu --set full --clock-control none --import-source on -s 7 -c 7 -o $out/chain \
  python bench.py --instances 200000 --steps 1 --warmup 1 --profile-run --no-secondary > $out/chain.log 2>&1
ls -la $out
