#!/bin/bash
# A/B: the kernel lab on _old_tree (previous build) vs the current tree
(cd _old_tree && python lab_sddmm_tma.py 2>&1 | grep -v Warn | sed 's/^/OLD /')
python scripts/lab_sddmm_tma.py 2>&1 | grep -v Warn | sed 's/^/NEW /'
