#!/usr/bin/env python
"""bench.py -- geometry-embed throughput on B200 (BASELINE.json metric:
"geometry-embed time (ms) & cells classified/s").

One step = one full embed_geometry (bins -> voxelization -> near-wall
refinement/octree split -> boundary cells -> cut-link LUT) of the workload's
synthetic mesh, inputs resident in HBM.  Default workload is BASELINE configs[1]
(C2: 112,000-face torus, N_x=64, L_max=4, 1 GPU).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config c2|c1|c4]
  python bench.py --impl reference ...   # CPU oracle port on the host cores

Multi-GPU (torchrun, one process per GPU): each rank embeds its own rigidly
translated copy of the mesh (independent objects, no data-path collective),
"scaling": "weak"; value = cells of all ranks / max-over-ranks time.
"""
import argparse
import json
import os
import subprocess
import sys
import tempfile
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

WORKLOADS = {
    "c1": dict(desc="C1: icosphere k=5 (20,480 faces), N_x=64, L_max=3", kind="sphere", sub=5,
               n_x=64, l_max=3),
    "c2": dict(desc="C2: torus 280x200 (112,000 faces), N_x=64, L_max=4", kind="torus", m=280, n=200,
               n_x=64, l_max=4),
    "c4": dict(desc="C4: torus 3000x1200 (7,200,000 faces), N_x=64, L_max=5", kind="torus", m=3000,
               n=1200, n_x=64, l_max=5),
    # C3: sphere D_s = 1/64 (icosphere k=5) in a 128^3 root, L_max=3, Re=20,
    # u_in=0.05: the embed plus the LUT consumer's
    # collide/stream step per level
    "c3": dict(desc="C3: sphere D=1/64 (icosphere k=5, 20,480 faces), N_x=128, L_max=3, Re=20 LBM",
               kind="sphere", sub=5, diameter=1.0 / 64, n_x=128, l_max=3, lbm=True),
}
METRIC = "geometry-embed cells classified/s"
UNIT = "cells/s"


def make_mesh(w, rank):
    from paper_2512_01251_b200 import make_icosphere, make_torus
    from paper_2512_01251_b200.mesh import translate
    m = (make_icosphere((0.5, 0.5, 0.5), w.get("diameter", 0.5), w["sub"]) if w["kind"] == "sphere"
         else make_torus(w["m"], w["n"]))
    if rank:
        rng = np.random.default_rng(rank)
        m = translate(m, (rng.random(3) - 0.5) / 64.0)
    return m


def make_cfg(w):
    from paper_2512_01251_b200 import EmbedConfig
    return EmbedConfig(n_x=w["n_x"], l_max=w["l_max"], n_spec=2, d_spec=0.05)


class Clocks:
    """nvidia-smi sampler during the timed region (B200_PROFILING.md)."""

    def __init__(self, index):
        self.f = tempfile.NamedTemporaryFile("w+", suffix=".csv", delete=False)
        q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
             "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
        try:
            self.p = subprocess.Popen(["nvidia-smi", "-i", str(index), f"--query-gpu={q}",
                                       "--format=csv,noheader,nounits", "-lms", "200"],
                                      stdout=self.f, stderr=subprocess.DEVNULL)
        except OSError:
            self.p = None

    def stop(self):
        if self.p is None:
            return None
        self.p.terminate()
        try:
            self.p.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.p.kill()
        self.f.flush()
        rows = []
        with open(self.f.name) as fh:
            for line in fh:
                parts = [x.strip() for x in line.split(",")]
                if len(parts) >= 9:
                    rows.append(parts)
        os.unlink(self.f.name)
        if not rows:
            return None
        sm = [float(r[1]) for r in rows if r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in rows if r[2].replace(".", "").isdigit()]
        reasons = set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for r in rows:
            for nm, val in zip(names, r[5:9]):
                if val.strip().lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": float(np.median(sm)) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": sorted(reasons),
                "samples": len(rows)}


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return d.get("hbm_gbs", 6650.0), "measured"
    return 6650.0, "fallback (B200_PROFILING.md)"


def ncu_traffic(config, *kernels):
    """dram__bytes_read.sum + dram__bytes_write.sum per launch, summed over
    `kernels`, from the committed ncu --set full summary
    (profiles/ncu_traffic.json, written by tools/ncu_traffic.py), or None."""
    p = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if not os.path.exists(p):
        return None
    d = json.load(open(p)).get(config, {})
    if "k_lut_blocks" not in d:  # the capture must hold the LUT kernel at least
        return None
    # kernels absent from the capture did not run in it (e.g. no large faces
    # at C4: the warp-flattened enumeration is not launched with work)
    return float(sum(d[k]["dram_bytes"] for k in kernels if k in d))


def cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def cpu_baseline(mesh, cfg, cells, repeat=3):
    """The oracle port (the reference ships no implementation of this path)
    on all host cores: median of `repeat` full embeds; also returns the
    oracle's algorithmic operation counters."""
    from oracle import oracle as O
    O.build()
    thr = len(os.sched_getaffinity(0))
    O.set_threads(thr)
    fc, nrm = mesh.faces_coord, mesh.normals
    cap = cfg.block_capacity(float(mesh.face_areas().sum()))
    ts = []
    for _ in range(repeat):
        t0 = time.perf_counter()
        O.embed(fc, nrm, cfg, cap)
        ts.append(time.perf_counter() - t0)
    ops = O.op_counters()
    med_s = float(np.median(ts))
    return {"value": cells / med_s, "unit": UNIT, "cores": thr, "kind": "port", "cpu_model": cpu_model(),
            "sample": f"full embed of the same mesh, median of {repeat} runs: {med_s * 1e3:.1f} ms "
                      f"(min {min(ts) * 1e3:.1f})",
            "ms": med_s * 1e3}, ops


def fp_peaks():
    """Measured FP32 / FP64 instruction rates (tools/micro/fp_peak.cu on this
    pool's B200, profiles/fp_peaks.json): one counted op = one instruction."""
    p = os.path.join(ROOT, "profiles", "fp_peaks.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return d["fp32_add_tinstr"] * 1e12, d["fp64_add_tinstr"] * 1e12, "measured (profiles/fp_peaks.json)"
    # nominal: 148 SMs x 128 FP32 / 64 FP64 lanes x 1.965 GHz
    return 37.2e12, 18.6e12, "nominal"


def level_counts(eng, mesh, cfg):
    """Per-level counts behind the algorithmic bytes: blocks N_L, kept faces
    F_k,L and pairs P_L of the 1D bins, bin faces of the level's blocks W_L
    (sum over blocks of their bin's face count), through the SPEC API."""
    import torch
    from paper_2512_01251_b200 import binning
    g = eng.grid
    ls = g.level_starts()
    out = []
    for L in range(g.n_levels):
        s, e = int(ls[L]), int(ls[L + 1])
        bl = binning.build_level(mesh, L, cfg)
        Bx, By, _ = cfg.bins(L)
        co = g.coords[s:e].long()
        idx = co[:, 0] + Bx * (co[:, 1] + By * co[:, 2])
        W = int(bl.counts.long()[idx].sum().item())
        out.append({"level": L, "blocks": e - s, "kept_faces": int(bl.filter_map.compact_map.numel()),
                    "pairs": int(bl.counts.long().sum().item()), "bin_faces_of_blocks": W,
                    "bins": cfg.n_bins(L)})
        del bl
        torch.cuda.empty_cache()
    return out


def kernel_rooflines(kt, lv, cfg, F, n_b, stats, ops, hbm, fp32, fp64, traffic):
    """Per-kernel roofline entries: algorithmic bytes (SURVEY.md §8d
    formulas) and ops (the oracle's counters for the FP64
    stages, the enumeration's FP32 intersection tests) per embed, over the
    kernel's device time from the per-kernel CUDA events (kt: {name:
    (launches, ms)}); frac = max(bytes/t / HBM, ops/t / FP peak)."""
    Lf = len(lv) - 1
    N = [x["blocks"] for x in lv]
    nprop = cfg.n_prop
    P = [x["pairs"] for x in lv]            # (bin, face) pairs per level
    K = [x["kept_faces"] for x in lv]       # kept faces per level
    W = [x["bin_faces_of_blocks"] for x in lv]  # pairs whose bin holds a block
    # 1D indicators: face records read once, kept-face map entries written
    b_ind = F * 96 + sum(K) * 4
    # embed pairs: kept face ids + records read, (bin, face) pairs written
    b_pairs = sum(k * 100 + p * 8 for k, p in zip(K, P))
    # pairs -> blocks (K1) and the counting-sort scatter (K3)
    b_pblk = sum(p * (8 + 4) + n * 4 for p, n in zip(P, N))
    b_pscat = sum(p * (8 + 4) + w * 4 for p, w in zip(P, W))
    # scans: block-bin offsets, row order (2), adapt child ids, tables, cut-link parents
    parents = (cfg.nb[0] << Lf) * (cfg.nb[1] << Lf) * (cfg.nb[2] << Lf) // 8
    b_scan = sum(n * 12 * 4 for n in N) + N[Lf] * 12 + parents * 12
    b_vox = sum(n * 136 + w * 100 for n, w in zip(N, W))
    # sparse rows: masks read + written, the row order (ids, rows) read; the
    # next level's order written (ids + rows of its positions)
    b_rows = sum(n * (128 + 4 + 16) for n in N) + sum(N[L + 1] * 8 + N[L] * 12 for L in range(Lf))
    # per pass: the block's own 27-slot neighbour row and flag bytes (the
    # neighbours' flags are the same bytes re-read through L2, not HBM)
    b_mark = sum(N[L] * (27 * 4 + 2) * (nprop + 2) for L in range(Lf))
    b_adapt = sum(N[L + 1] * 304 + N[L] * 108 for L in range(Lf))
    # the neighbour row, the block's own solid word (the 26 neighbours' words
    # are L2 re-reads), masks read + written, count, flags
    b_bnd = N[Lf] * (27 * 4 + 8 + 64 + 64 + 4 + 2)
    lines, tests = stats["lines"], stats["tests"]
    links = 2 * lines  # <= 2 links per recorded line (q-records)
    # enumeration: face records read once, q-records written
    b_enum = F * 96 + lines * 16
    # parent buckets (counted as the records become q-records): q-records
    # read once, parent-ordered links written, the parent-key scan
    b_bucket = lines * 16 + links * 8 + parents * 12
    # LUT: every slot written once (6912 B), its links read
    b_lut = n_b * (27 * 64 * 4 + 4 + 16) + links * 8
    o = lambda k: ops.get(k, {}).get("sat_ops", 0) + ops.get(k, {}).get("other_ops", 0) if ops else None
    rows = [
        ("k_indicators_all", ["k_indicators_all"], b_ind, o("indicators"), "fp64",
         "1D ray indicators of every level + per-level kept-face maps, one pass over the 96-B face records; "
         "ops: the oracle's SAT ops"),
        ("k_pairs", ["k_pairs"], b_pairs, o("pairs"), "fp64",
         "Alg. 2 bin pairs of every level (compact append); ops: the oracle's per-candidate SAT ops"),
        ("k_pair_blocks", ["k_pair_blocks"], b_pblk, None, None, "pairs -> level-L blocks (forest descent) + counts"),
        ("k_pair_scatter", ["k_pair_scatter"], b_pscat, None, None, "counting-sort scatter into block bins"),
        ("scan_kernel", ["scan_kernel"], b_scan, None, None,
         "block-bin offsets, row order, child ids, tables, cut-link parent buckets"),
        ("k_voxelize", ["k_voxelize"], b_vox, o("voxelize"), "fp64",
         "Alg. 3, every level; ops: the oracle's slab-SAT ops + 4 x 11 per accepted (row, face)"),
        ("k_xrows", ["k_xrows", "k_rows_children", "k_rows_init"], b_rows, None, None,
         "Alg. 5 +-x over the sparse rows + finalize; next level's row order"),
        ("k_mark", ["k_mark_sb", "k_mark_adj", "k_mark_prop"], b_mark, None, None,
         "near-wall marking, (N_prop + 2) passes"),
        ("k_adapt", ["k_adapt_level", "k_adapt_children"], b_adapt, None, None, "refine-only adapt"),
        ("k_boundary", ["k_boundary"], b_bnd, None, None, "boundary cells (finest level)"),
        ("k_links_enum", ["k_links_small", "k_links_enum", "k_links_q"], b_enum, tests * 18 if tests else None,
         "fp32", "cut-link line enumeration -> q-records (exact FP64 q); ops: 18 FP32 ops per lattice line "
         "classified (3 edge functions + tests)"),
        ("k_link_buckets", ["k_block_scatter"], b_bucket, None, None,
         "links scattered into finest-parent-key buckets (the counts are made in the enumeration)"),
        ("k_lut_blocks", ["k_lut_blocks", "k_links_band", "k_links_ovf", "k_links_full"], b_lut, None, None,
         "LUT slots written once from shared memory (-1 + min-merged links); exact band / overflow paths"),
    ]
    out = []
    for name, ks, nbytes, nops, pipe, note in rows:
        ms = sum(kt[k][1] for k in ks if k in kt)
        launches = sum(kt[k][0] for k in ks if k in kt)
        if ms <= 0:
            continue
        gbs = nbytes / (ms / 1e3) / 1e9
        e = {"kernel": name, "launches_per_embed": launches, "ms_per_embed": ms,
             "algorithmic_bytes": int(nbytes), "achieved_gbs": gbs, "hbm_frac": gbs / hbm,
             # ncu DRAM bytes per launch x this embed's launches of each kernel
             "traffic": (sum(traffic[k]["dram_bytes"] * kt[k][0] for k in ks if k in traffic and k in kt)
                         if traffic else None), "note": note}
        if nops:
            peak = fp64 if pipe == "fp64" else fp32
            rate = nops / (ms / 1e3)
            e.update({"algorithmic_ops": int(nops), "ops_pipe": pipe, "achieved_tops": rate / 1e12,
                      "ops_frac": rate / peak})
        # every kernel of the path is bounded by HBM bytes or by latency /
        # issue (none is a dense FP pipe workload): frac is the HBM fraction.
        # ops_frac is context: for the FP64 stages it counts the ORACLE's
        # exact SAT work (>1 = the FP32 classifiers skip that much of it), for
        # the enumeration the FP32 intersection tests actually executed
        e["bound"], e["frac"] = "hbm", e["hbm_frac"]
        out.append(e)
    return out


def ncu_kernel_traffic(config):
    """Per-kernel DRAM bytes (dram__bytes_read.sum + dram__bytes_write.sum)
    per launch (mean over the captured launches) from the committed ncu --set
    full summary, or None."""
    p = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if not os.path.exists(p):
        return None
    d = json.load(open(p)).get(config)
    if not d:
        return None
    k = dict(d.get("kernels", {}))
    # kernel-timer names (check_launch) that differ from the device symbols
    for kt_name, sym in (("k_pairs", "k_pairs_append"), ("k_adapt_children", "k_adapt_children_t"),
                         ("k_links_small", "k_links_smallq")):
        if sym in k:
            k[kt_name] = k[sym]
    return k


def dist_setup():
    import torch
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if ws > 1:
        import torch.distributed as dist
        # VF_BENCH_BACKEND=gloo: exercise the multi-rank path on one GPU (tests)
        backend = os.environ.get("VF_BENCH_BACKEND") or ("nccl" if torch.cuda.is_available() else "gloo")
        if torch.cuda.is_available():
            torch.cuda.set_device(local % torch.cuda.device_count())
        dist.init_process_group(backend)
    return ws, rank, local


def barrier(ws):
    if ws > 1:
        import torch.distributed as dist
        dist.barrier()


def allmax(ws, x):
    if ws <= 1:
        return x
    import torch
    import torch.distributed as dist
    t = torch.tensor([x], dtype=torch.float64, device="cuda" if torch.cuda.is_available() else "cpu")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def run_reference(args, w, ws, rank):
    """--impl reference: the CPU oracle port (the reference ships no
    implementation of this path) timed on the host cores, rank 0 only."""
    if rank != 0:
        return
    from oracle import oracle as O
    O.build()
    thr = len(os.sched_getaffinity(0))
    O.set_threads(thr)
    mesh = make_mesh(w, 0)
    cfg = make_cfg(w)
    fc, nrm = mesh.faces_coord, mesh.normals
    cap = cfg.block_capacity(float(mesh.face_areas().sum()))
    for _ in range(args.warmup):
        r = O.embed(fc, nrm, cfg, cap)
    cells = None
    t0 = time.perf_counter()
    for _ in range(args.steps):
        r = O.embed(fc, nrm, cfg, cap)
    dt = time.perf_counter() - t0
    cells = 64 * r.grid.n_used
    value = cells * args.steps / dt
    line = {"metric": METRIC, "value": value, "unit": UNIT, "impl": "reference", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": dt / args.steps * 1e3,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic",
            "config": {"workload": w["desc"], "cells_per_embed": cells, "faces": int(mesh.n_faces)},
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": thr, "kind": "port",
                             "sample": f"full embed per step x {args.steps}"},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def lbm_block(eng, w, args, flush):
    """C3: the LUT consumer on the embedded grid.  Per level one BGK
    collide/stream step (csrc/vf_lbm.cu; IBB walls from the LUT on the finest
    level, SBB below), timed with CUDA events, and one coarse step of the
    nested hierarchy (solver.step_hierarchy, interface exchange included).
    Embed overhead = embed time / coarse step."""
    import torch
    from paper_2512_01251_b200.solver import FlowConfig, LbmLevel
    grid, table = eng.run()
    Lf = grid.n_levels - 1
    D_f = w["diameter"] * 4 * w["n_x"] // 4 * 2 ** Lf  # sphere diameter in finest cells
    peak, peak_kind = peaks()
    levels = []
    coarse_ms = 0.0
    for L in range(grid.n_levels):
        s, e = grid.level_range(L)
        flow = FlowConfig(Re=20.0, u_in=0.05, D_s=D_f / 2 ** (Lf - L),
                          bc_scheme="IBB" if L == Lf else "SBB")
        lv = LbmLevel(grid, L, table if L == Lf else None, flow).init_equilibrium(1.0, (0.05, 0, 0))
        for _ in range(3):
            lv.step(1, force=False)
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        k = max(args.steps, 10)
        flush.fill_(1.0)
        a.record()
        lv.step(k, force=(L == Lf))
        b.record()
        torch.cuda.synchronize()
        ms = a.elapsed_time(b) / k
        cells = (e - s) * 64
        nbytes = cells * (27 * 4 * 2 + 1)
        levels.append({"level": L, "blocks": e - s, "cells": cells, "tau": flow.tau,
                       "step_ms": ms, "cell_updates_per_s": cells / (ms / 1e3),
                       "hbm_gbs": nbytes / (ms / 1e3) / 1e9, "hbm_frac": nbytes / (ms / 1e3) / 1e9 / peak})
        coarse_ms += 2 ** L * ms
        if L == Lf:
            drag = lv.force.cpu().numpy() / k
    # one coarse step of the nested hierarchy (step_hierarchy: level L takes
    # 2^L substeps, cubic ghost fill before each fine substep, restriction
    # after), replayed from a CUDA graph of two coarse steps
    from paper_2512_01251_b200.solver import LbmHierarchy
    flow0 = FlowConfig(Re=20.0, u_in=0.05, D_s=D_f / 2 ** Lf, bc_scheme="IBB")
    h = LbmHierarchy(grid, table, flow0, order=3).init_equilibrium(1.0, (0.05, 0, 0))
    gr = h.graph()
    for _ in range(2):
        gr.replay()
    torch.cuda.synchronize()
    k = max(args.steps // 2, 5)
    flush.fill_(2.0)
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(k):
        gr.replay()
    b.record()
    torch.cuda.synchronize()
    hier_ms = a.elapsed_time(b) / (2 * k)
    return {"levels": levels, "coarse_step_ms": hier_ms, "coarse_step_ms_levels_only": coarse_ms,
            "taus": h.taus, "wall_force_lattice": [float(x) for x in drag],
            "note": "per level: one BGK collide/stream (f32 SoA, 216 B/cell algorithmic), IBB from the LUT; "
                    "coarse_step_ms = one step_hierarchy coarse step (2^L substeps per level, cubic ghost "
                    "fill + restriction between levels, CUDA graph); coarse_step_ms_levels_only = "
                    "sum_L 2^L t_L without the exchange",
            "peak_kind": peak_kind}


def pipelined_e2e(eng, mesh, cfg, verts, fidx, steps, ws, holder):
    """Total device time of `steps` pipelined end-to-end embeds (two engines
    alternating, H2D / D2H on their own streams), max over ranks.  Each step:
    H2D of the indexed mesh (vertices + faces_indexed, pinned), face records
    and normals on the device, embed, sparse LUT, D2H of grid + cut links."""
    import torch
    from paper_2512_01251_b200.voxelizer import EmbedEngine
    eng2 = EmbedEngine(mesh, cfg, capacity=eng.grid.capacity)
    eng2.run()
    engines = [eng, eng2]
    s_in, s_out = torch.cuda.Stream(), torch.cuda.Stream()
    outs = [None, None]

    def go(k):
        e = engines[k % 2]
        outs[k % 2], holder["h2d"], holder["d2h"] = e.embed_indexed_async(verts, fidx, outs[k % 2], s_in, s_out)

    for k in range(4):  # warm-up (allocates the pinned outputs)
        go(k)
    torch.cuda.synchronize()
    barrier(ws)
    cur = torch.cuda.current_stream()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(cur)
    for s_ in (s_in, s_out, eng.stream, eng2.stream):
        s_.wait_event(a)
    for k in range(steps):
        go(k)
    cur.wait_stream(s_out)
    b.record(cur)
    torch.cuda.synchronize()
    barrier(ws)
    for e in engines:
        e.check_async()
    return allmax(ws, a.elapsed_time(b))


def timed_steps(run, steps, flush, ws):
    """Barrier + sync, then `steps` runs each bracketed by CUDA events on the
    current stream (the L2 flush between steps stays outside the events);
    returns the per-step device times (ms) of this rank."""
    import torch
    starts = [torch.cuda.Event(enable_timing=True) for _ in range(steps)]
    ends = [torch.cuda.Event(enable_timing=True) for _ in range(steps)]
    barrier(ws)
    torch.cuda.synchronize()
    for k in range(steps):
        flush.fill_(float(k))
        starts[k].record()
        run()
        ends[k].record()
    torch.cuda.synchronize()
    barrier(ws)
    return [a.elapsed_time(b) for a, b in zip(starts, ends)]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="c4", choices=sorted(WORKLOADS))
    ap.add_argument("--mode", default="shard", choices=["shard", "objects"],
                    help="N>1: block-shard ONE mesh (strong scaling, NCCL flag exchange) or "
                         "embed independent translated copies (weak scaling, no collective)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    w = WORKLOADS[args.config]
    ws, rank, local = dist_setup()
    if args.impl == "reference":
        run_reference(args, w, ws, rank)
        barrier(ws)
        return

    import torch
    from paper_2512_01251_b200 import _lib
    from paper_2512_01251_b200.voxelizer import EmbedEngine
    lib = _lib.require_cuda()
    dev = torch.cuda.current_device()
    sharded = ws > 1 and args.mode == "shard"
    mesh = make_mesh(w, 0 if sharded else rank)
    cfg = make_cfg(w)
    if sharded:
        from paper_2512_01251_b200.parallel import ShardedEmbed
        eng = ShardedEmbed(mesh, cfg)
        run = eng.run
    else:
        eng = EmbedEngine(mesh, cfg)
        run = eng.run  # one embed (CUDA graph or eager) + one host sync (status, N_b)
    for _ in range(args.warmup):
        run()
    torch.cuda.synchronize()
    flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device="cuda")
    # clocks: sample a ~1 s load phase of the same step plus the timed region
    clocks = Clocks(dev)
    t_load = time.perf_counter()
    while time.perf_counter() - t_load < 1.0:
        run()
    torch.cuda.synchronize()
    launches0 = lib.vf_launch_count()
    if sharded:
        step_ms = timed_steps(run, args.steps, flush, ws)
    else:
        # steady state: embeds enqueued back to back on the engine stream
        # (no host sync per embed, so the host's launch work overlaps the
        # previous embed); each step's events bracket exactly its embed
        # (engine stream after the flush, current stream after the embed);
        # status and N_b of every step validated after the timed region
        cur = torch.cuda.current_stream()

        def run_pipelined():
            eng.stream.wait_stream(cur)
            eng.run_async()
            cur.wait_stream(eng.stream)

        step_ms = timed_steps(run_pipelined, args.steps, flush, ws)
        eng.check_async()
    launches = lib.vf_launch_count() - launches0
    ck = clocks.stop()
    total_ms = allmax(ws, float(sum(step_ms)))
    cells = eng.cells_classified()
    if sharded:
        cells_all = cells  # one mesh: every rank reports the same grid
    else:
        cells_all = cells
        if ws > 1:
            import torch.distributed as dist
            t = torch.tensor([cells], dtype=torch.float64, device="cuda")
            dist.all_reduce(t)
            cells_all = int(t.item())
    value = cells_all * args.steps / (total_ms / 1e3)
    g = eng.grid
    med = lambda a: float(np.median(a))
    F = eng.mesh.n_faces
    peak, peak_kind = peaks()
    stages, roofline, kernels_per_step = None, None, launches // max(args.steps, 1)
    per_kernel = None
    if not sharded:
        n_b = int(eng.n_b_host[0])
        # kernels per step: count one eager (non-graph) embed
        l0 = lib.vf_launch_count()
        eng.run(timed=True)
        kernels_per_step = lib.vf_launch_count() - l0
        # the cut-link kernels timed alone (enumeration serial on the main
        # stream, so its events are not stretched by the overlapped level
        # pipeline) -- the roofline figure; the overlapped time is reported too
        stage, link_ms, link_ovl = [], [], []
        old_serial = lib.vf_set_serial_links(1)
        try:
            for k in range(max(3, min(args.steps, 5))):
                flush.fill_(float(k))
                eng.run(timed=True)
                torch.cuda.synchronize()
                stage.append(eng.timings())
                link_ms.append(eng.link_kernel_ms())
        finally:
            lib.vf_set_serial_links(old_serial)
        for k in range(3):
            flush.fill_(float(k))
            eng.run(timed=True)
            torch.cuda.synchronize()
            link_ovl.append(eng.link_kernel_ms())
        stages = {k: med([getattr(s, k) for s in stage]) for k in
                  ("binning", "voxelization", "refinement", "boundary", "links", "total")}
        # per-kernel device times: every kernel of one eager embed on the
        # engine stream in order, CUDA events after each launch (median of 3)
        kts = [eng.kernel_times() for _ in range(3)]
        kt = {k: (kts[0][k][0], med([x[k][1] for x in kts if k in x])) for k in kts[0]}
        link_stats = eng.link_stats()
        # the cut-link group: algorithmic bytes = the face
        # records read once (96 B/face) + the LUT of the mapped blocks written
        # once (27 x 64 x 4 = 6912 B per boundary block); the group's kernels
        # write each LUT slot exactly once (no separate -1 fill)
        link_bytes = F * 96 + n_b * 27 * 64 * 4
        lk = med(link_ms)
        achieved = link_bytes / (lk / 1e3) / 1e9
        roofline = {"kernel": "cut-link group", "bound": "hbm", "achieved": achieved, "peak": peak,
                    "peak_kind": peak_kind, "unit": "GB/s", "frac": achieved / peak,
                    "traffic": ncu_traffic(args.config, "k_links_smallq", "k_links_enum", "k_links_q",
                                           "k_block_scatter", "k_lut_blocks"),
                    "kernel_ms": lk, "algorithmic_bytes": int(link_bytes),
                    "kernel_ms_overlapped": med(link_ovl),
                    "timed": "CUDA events around the cut-link kernels run alone (vf_set_serial_links): "
                             "the grid-independent line enumeration with its exact q and parent bucketing, "
                             "then the LUT kernel after the tables (writes every slot's 6912 B once); "
                             "kernel_ms_overlapped = the same events in the production schedule"}
    else:
        n_b = int(run()[1].n_b)

    lbm = lbm_block(eng, w, args, flush) if (w.get("lbm") and not sharded) else None
    if lbm:
        lbm["embed_ms"] = med(step_ms)
        lbm["embed_over_coarse_step"] = med(step_ms) / lbm["coarse_step_ms"]

    e2e = None
    if not args.no_e2e:
        fc = torch.from_numpy(np.ascontiguousarray(mesh.faces_coord)).pin_memory() if sharded else None
        nr = torch.from_numpy(np.ascontiguousarray(mesh.normals)).pin_memory() if sharded else None
        if sharded:
            dfc = torch.empty((F, 9), dtype=torch.float64, device="cuda")
            dn = torch.empty((F, 3), dtype=torch.float64, device="cuda")
            holder = {}

            def e2e_step():
                dfc.copy_(fc, non_blocking=True)
                dn.copy_(nr, non_blocking=True)
                _lib.check(lib.vf_pack_faces(_lib.ptr(dfc), _lib.ptr(dn), F, _lib.ptr(eng.mesh.faces),
                                             _lib.stream_ptr()))
                gg, tt = eng.run()
                n = gg.n_used
                outs = [gg.coords[:n], gg.nbr[:n], gg.child[:n], gg.bflags[:n], gg.masks[:n],
                        tt.contraction_map[:n], tt.lengths]
                d2h = 0
                for i, t_ in enumerate(outs):
                    buf = holder.get(i)
                    if buf is None or buf.shape != t_.shape:
                        buf = holder[i] = torch.empty(t_.shape, dtype=t_.dtype).pin_memory()
                    buf.copy_(t_, non_blocking=True)
                    d2h += t_.numel() * t_.element_size()
                holder["d2h"] = d2h
        else:
            holder = {"out": None}

            def e2e_step():
                holder["out"], h2d_, holder["d2h"] = eng.embed_host(fc, nr, holder["out"])
        if not sharded:
            # pipelined serving: two engines alternate so that one step's D2H
            # (PCIe-bound) overlaps the next step's H2D + embed; every step
            # uploads the indexed mesh and downloads the grid + the cut links
            verts = torch.from_numpy(np.ascontiguousarray(mesh.vertices, dtype=np.float64)).pin_memory()
            fidx = torch.from_numpy(np.ascontiguousarray(mesh.faces_indexed, dtype=np.int32)).pin_memory()
            e2e_ms = pipelined_e2e(eng, mesh, cfg, verts, fidx, args.steps, ws, holder)
        else:
            for _ in range(2):
                e2e_step()
            e2e_ms = allmax(ws, float(sum(timed_steps(e2e_step, args.steps, flush, ws))))
        e2e = {"value": cells_all * args.steps / (e2e_ms / 1e3), "unit": UNIT,
               "h2d_bytes_per_step": int(holder.get("h2d", F * 96)), "d2h_bytes_per_step": int(holder["d2h"]),
               "ms_per_step": e2e_ms / args.steps,
               "mode": ("pipelined (EmbedEngine.embed_indexed_async, two engines alternating): each step "
                        "uploads the mesh as the reference TriangleMesh's vertices (V,3) f64 + faces_indexed "
                        "(F,3) int32 from pinned memory, builds the face records and unit normals on the "
                        "device (np.cross/norm bit for bit), embeds, and downloads the grid (coords, nbr, "
                        "child, bflags, masks, contraction map) and the LUT's cut links as (flat index, q) "
                        "pairs (the -1 entries implicit); D2H of step k overlaps H2D/embed of step k+1"
                        if not sharded else "sequential: faces + normals up, grid + dense LUT down")}

    if rank != 0:
        return
    cpu, ops = None, None
    if not args.no_cpu_baseline and ws == 1:
        cpu, ops = cpu_baseline(mesh, cfg, cells, repeat=3 if F > 1_000_000 else 10)
    if not sharded:
        fp32, fp64, fp_kind = fp_peaks()
        lv = level_counts(eng, mesh, cfg)
        per_kernel = kernel_rooflines(kt, lv, cfg, F, n_b, link_stats, ops, peak, fp32, fp64,
                                      ncu_kernel_traffic(args.config))
        dom = max(per_kernel, key=lambda e: e["ms_per_embed"])
        roofline = {"kernel": dom["kernel"], "bound": "hbm", "achieved": dom["achieved_gbs"], "peak": peak,
                    "peak_kind": peak_kind, "unit": "GB/s", "frac": dom["frac"],
                    "traffic": dom["traffic"], "kernel_ms": dom["ms_per_embed"],
                    "algorithmic_bytes": dom["algorithmic_bytes"],
                    "algorithmic_ops": dom.get("algorithmic_ops"),
                    "timed": "the dominant kernel (largest device time per embed) from per-kernel CUDA events "
                             "of one eager embed with every kernel on one stream (vf_ktimer); roofline.kernels "
                             "holds every kernel: frac = algorithmic bytes/t / measured HBM copy peak; ops_frac "
                             "= algorithmic ops/t / measured FP32 or FP64 instruction rate (context)",
                    "links_group": roofline, "level_counts": lv, "link_stats": link_stats,
                    "fp_peaks_tops": {"fp32": fp32 / 1e12, "fp64": fp64 / 1e12, "kind": fp_kind},
                    "kernels": per_kernel}
    par = "single GPU"
    if ws > 1:
        par = (f"block-sharded x{ws} (row ownership, NCCL all-reduce of per-level flags, "
               f"finest solid masks and boundary counts)" if sharded else f"independent objects x{ws}")
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": ws, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": total_ms / args.steps, "higher_is_better": True,
        "scaling": "strong" if sharded else "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic",
        "config": {"workload": w["desc"], "faces": int(F), "cells_per_embed": int(cells),
                   "blocks": int(g.n_used), "boundary_blocks": n_b,
                   "embed_ms_median": med(step_ms), "stage_ms_serial": stages,
                   "l2": "64 Mi-float (256 MB) buffer rewritten between steps, outside step events",
                   "step": ("one sharded embed + its host syncs" if sharded else
                            "one embed; embeds enqueued back to back on the engine stream (no host sync "
                            "per embed), each step's CUDA events bracketing its embed, status / N_b "
                            "validated after the timed region"),
                   "parallelism": par},
        "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e, "lbm": lbm,
        "gpu_launches": int(kernels_per_step * args.steps),
        "gpu_launch_note": (f"{kernels_per_step} kernels per embed" +
                            ("" if sharded else (", issued as one CUDA graph per step" if eng.use_graph
                                                  else ", eager launches (stream priorities)"))),
        "clocks": ck,
    }
    print(json.dumps(line), flush=True)


if __name__ == "__main__":
    main()
