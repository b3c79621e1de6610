for g in 32 16 8; do echo "== G=$g" >> gpurun_out/p_imp.txt; GSB_IMP_G=$g python tools/attrib.py 0 | grep -E "importance|step" >> gpurun_out/p_imp.txt; done
