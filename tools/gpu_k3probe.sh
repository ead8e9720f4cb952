#!/bin/bash
# K3 A/B without the whole-prefill timing in front (power state), clocks sampled while timing.
timeout 900 python tools/k3_ab.py 4 2>&1 | tail -12
