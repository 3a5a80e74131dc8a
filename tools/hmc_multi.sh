O=gpurun_out/ab75; mkdir -p $O
for i in 1 2; do for v in mm24 mm12; do SPECWALK_LIB=$PWD/paper_2010_03817_b200/libspecwalk_$v.so python tools/probe_hmc.py 20:20:16384:3 16:16:16384:3 2>/dev/null | sed "s/^/$v /" >> $O/hmc.txt; done; done
