#!/bin/bash
# same-box A/B of build_ab/*.so on the given workloads
for w in "$@"; do for v in $(ls build_ab | sed 's/.so//'); do echo "$v $w"; python tools/ab_lib.py build_ab/$v.so $w > /tmp/o.txt 2>&1; grep -v stress /tmp/o.txt | head -3; done; done
nvidia-smi --query-gpu=clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active --format=csv
