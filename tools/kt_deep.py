"""Per-kernel device times (vf_ktimer, one eager embed, all kernels on one
stream) of the 7.2M-face torus at a given L_max: python tools/kt_deep.py 7"""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2512_01251_b200 import EmbedConfig, make_torus  # noqa: E402
from paper_2512_01251_b200.voxelizer import EmbedEngine  # noqa: E402
lm = int(sys.argv[1]) if len(sys.argv) > 1 else 7
eng = EmbedEngine(make_torus(3000, 1200), EmbedConfig(n_x=64, l_max=lm))
for _ in range(2):
    eng.run()
kt = eng.kernel_times()
tot = sum(v[1] for v in kt.values())
print(json.dumps({"l_max": lm, "total_ms": tot}))
for k, v in sorted(kt.items(), key=lambda kv: -kv[1][1])[:25]:
    print(f"{k:28s} {v[0]:4d} {v[1]:.4f}")
