#!/bin/bash
# castscale variants at N=1 (run on the GPU box)
for V in 4x256x4 8x256x4 2x256x8 4x512x2 8x512x2 4x128x8 8x256x2 4x256x8; do
  echo "$V $(TORUS_CS=$V timeout 120 python bench.py --steps 200 --no-cpu --no-e2e | tail -1 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["us_per_call"],2), round(d["roofline"]["frac"],3))')"
done
