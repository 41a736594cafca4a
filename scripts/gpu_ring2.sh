#!/bin/bash
for c in 16 24 32 48 64; do
  timeout 60 python bench.py --cells $c --steps 20 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ring_c$c.log 2>&1
  echo "cells=$c rc=$? $(tail -1 gpurun_out/ring_c$c.log | cut -c1-120)"
done
