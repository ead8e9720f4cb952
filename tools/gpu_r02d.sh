#!/bin/bash
bash tools/gpu_fqkv.sh
bash tools/gpu_ncu_r02.sh
