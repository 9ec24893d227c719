#!/bin/bash
for a in 1 5 6 8; do for b in 1 5 6; do DD_SPMV_MINB_1=$a DD_SPMV_MINB_2=$b timeout -s KILL 120 python tools/solve_probe.py; done; done
