#!/bin/bash
export CKV_LIB=$PWD/paper_2412_03213_b200/libckv_b200_seldbg.so
CKV_DEBUG_TIMING=1 timeout 300 python tools/layer_prof.py 2 8 2>&1 | grep "k_select_fused dbg" | tail -40 | sort | uniq -c | sort -rn | head -8
