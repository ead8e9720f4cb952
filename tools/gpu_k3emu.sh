#!/bin/bash
timeout 1500 python tools/k3_ab.py 4 4096 "base:" "emu1:PSK_LIB=paper_2602_12029_b200/var_emu1.so" "emu2:PSK_LIB=paper_2602_12029_b200/var_emu2.so" 2>&1 | tail -16
