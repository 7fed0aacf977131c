import os, sys, json
os.environ["VF_KT_EACH"]="1"
sys.path.insert(0,'/root/repo')
import bench
from paper_2512_01251_b200.voxelizer import EmbedEngine
c=sys.argv[1]
w=bench.WORKLOADS[c]; eng=EmbedEngine(bench.make_mesh(w,0), bench.make_cfg(w))
for _ in range(3): eng.run()
kt=eng.kernel_times()
for k,v in kt.items(): print(k, round(v[1],4))
print("levels", eng.grid.level_starts()[:eng.grid.n_levels+1].tolist())
