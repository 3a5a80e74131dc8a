import os, sys
sys.path.insert(0, ".")
import paper_2010_03817_b200 as sw, specgen
os.environ["SPECWALK_DEBUG_VOLUME"] = "1"
S = sw.Spectrahedron.from_instance(specgen.rand_cube(12, 12, 2))
try:
    print(S.volume(0.1, 0, 256, walk_len=5, burn=20))
except Exception as e:
    print("ERR", e)
