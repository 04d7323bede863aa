#!/bin/bash
# A/B of built libraries at 1M M5: tools/ab_libs.sh rounds a.so b.so ...
R=$1; shift
for r in $(seq 1 $R); do bash tools/ab_stages.sh "$@"; done
