"""STL ingestion throughput: GPU parse_stl (text
bytes on the host -> TriangleMesh with host arrays + device face records) vs
the reference parse_stl (pure Python, timed only where /root/reference
exists, i.e. the build container).

  python tools/bench_stl.py [c2|c4] [--reference]"""
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def stl_bytes(fc):
    # "%.9e" coordinates (round-trip-ish, typical of exporters)
    v = fc.reshape(-1, 3)
    verts = ["      vertex {:.9e} {:.9e} {:.9e}".format(*p) for p in v]
    out = ["solid bench"]
    for f in range(len(fc)):
        out += ["  facet normal 0 0 0", "    outer loop", verts[3 * f], verts[3 * f + 1], verts[3 * f + 2],
                "    endloop", "  endfacet"]
    out.append("endsolid bench")
    return ("\n".join(out) + "\n").encode()


def main():
    which = sys.argv[1] if len(sys.argv) > 1 and not sys.argv[1].startswith("-") else "c2"
    from paper_2512_01251_b200 import make_torus
    mesh = make_torus(280, 200) if which == "c2" else make_torus(3000, 1200)
    data = stl_bytes(mesh.faces_coord)
    line = {"workload": f"{which}: torus, {mesh.n_faces} faces, {len(data) / 1e6:.1f} MB ASCII STL"}
    if "--reference" in sys.argv:
        import importlib.util
        spec = importlib.util.spec_from_file_location("vref_geometry", "/root/reference/pkg/src/voxforest/geometry.py")
        geo = importlib.util.module_from_spec(spec)
        sys.modules["vref_geometry"] = geo
        spec.loader.exec_module(geo)
        sample = 20000 if mesh.n_faces > 20000 else mesh.n_faces
        sdata = stl_bytes(mesh.faces_coord[:sample])
        t0 = time.perf_counter()
        geo.parse_stl(sdata)
        dt = time.perf_counter() - t0
        line["reference"] = {"faces_per_s": sample / dt, "sample_faces": sample, "sample_s": dt,
                             "cores": 1, "cpu": "build container (Intel Xeon), pure-Python parser"}
    else:
        import torch
        from paper_2512_01251_b200 import stl
        for _ in range(2):
            stl.parse_stl(data)
        torch.cuda.synchronize()
        ts = []
        for _ in range(5):
            t0 = time.perf_counter()
            m = stl.parse_stl(data)
            torch.cuda.synchronize()
            ts.append(time.perf_counter() - t0)
        t = float(np.median(ts))
        line["gpu"] = {"e2e_ms": t * 1e3, "faces_per_s": mesh.n_faces / t, "bytes_per_s": len(data) / t,
                       "n_verts": int(len(m.vertices)),
                       "note": "host bytes -> pinned -> HBM, tokenize/grammar/float/weld/normals on the "
                               "GPU, host arrays back (wall clock, median of 5)"}
    print(json.dumps(line))


if __name__ == "__main__":
    main()
