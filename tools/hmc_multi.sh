O=gpurun_out/ab72; mkdir -p $O
for i in 1 2; do for v in h5 h10 h15; do SPECWALK_LIB=$PWD/paper_2010_03817_b200/libspecwalk_$v.so python tools/probe_hmc.py 100:100:16384:1 72:72:16384:1 2>/dev/null | sed "s/^/$v /" >> $O/hmc.txt; done; done
