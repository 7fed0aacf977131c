/*
 * voxforest_b200.h -- C-ABI of the B200 geometry-embedding engine
 * (libvoxforest_b200.so, hand-written sm_100a CUDA).
 *
 * The reference (arxiv 2512.01251, /root/reference) has no FFI: its operator
 * API is the SPEC op set in the voxforest.binning / .forest / .voxelizer module
 * namespaces (only geometry.py/lattice.py ship as code).  Each
 * entry point below replaces one of those ops; the Python package
 * paper_2512_01251_b200 binds them with ctypes under the SPEC names (see
 * INTEGRATION.md).
 *
 * Conventions:
 *   - every pointer argument named d_* is DEVICE memory owned by the caller;
 *     the library keeps no pointer past the call and never frees caller memory.
 *   - sizes are int64_t; level descriptors are the POD vf_config below.
 *   - all calls are asynchronous and ordered on the given cudaStream_t
 *     (passed as void*); device-resident counts (d_level_start, d_count ...)
 *     are read by kernels, never by the host, so a level needs no host sync.
 *   - scratch is a caller-allocated workspace sized by the *_workspace_size
 *     call (CUB-style two-phase).
 *   - return value: VF_OK or a status code; message in vf_last_error()
 *     (thread-local).  Device-detected conditions (capacity exhausted, N_lim
 *     cap violated) are latched in the grid's d_status word and reported by
 *     vf_check_status().
 *   - results never depend on launch configuration or scheduling
 *     (SPEC.md:97,172,370,552): atomics are used only for order-free
 *     reductions (histograms, min), bins are re-sorted by face id.
 */
#ifndef VOXFOREST_B200_H
#define VOXFOREST_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define VF_ABI_VERSION 6
#define VF_MAX_LEVELS 16

/* status codes (SURVEY.md §8b "Errors") */
enum {
    VF_OK = 0,
    VF_EARG = 1,       /* bad argument                                      */
    VF_ECAPACITY = 2,  /* forest / pair capacity exhausted */
    VF_ENLIM = 3,      /* N_lim pair cap violated               */
    VF_ECUDA = 4,      /* CUDA error                                         */
    VF_ENCCL = 5,      /* NCCL error (multi-GPU path)                        */
    VF_EMESH = 6       /* invalid mesh: face index out of range / degenerate face (MeshError) */
};

/* cell mask enum (SPEC.md:197 cell_mask values) */
enum { VF_FLUID = 0, VF_SOLID = 1, VF_GUARD = 2, VF_GHOST = 3,
       VF_INTERFACE = 4, VF_BOUNDARY = 5 };
/* block flag bits (SPEC.md:197 block mask) */
enum { VF_BF_SOLID = 1, VF_BF_SB = 2, VF_BF_SA = 4, VF_BF_MARK = 8,
       VF_BF_REFINED = 16, VF_BF_BOUNDARY = 32 };
/* negative neighbour codes */
enum { VF_NB_OUTSIDE = -1, VF_NB_MISSING = -2, VF_NB_SOLID_NBR = -3 };

/* Level descriptor / embed config (SPEC.md:277-280 VoxelConfig + PAPER.md:291) */
typedef struct {
    int32_t nb[3];        /* root blocks per axis N_B                       */
    int32_t l_max;        /* grid levels                                    */
    int32_t n_spec;       /* N_spec                                         */
    int32_t n_prop;       /* N_prop                          */
    double  dx0;          /* root cell spacing                              */
    double  len[3];       /* domain lengths (origin 0)                      */
    double  eps_slab;
    double  eps_parallel; /* geometry.py:25                                 */
    /* block sharding (multi-GPU): x-runs never cross ranks because whole
     * level-L block rows (j,k) are owned.  0/1 = all.  With d_row_owner set,
     * rank = d_row_owner[row_base(L) + j + B_L,y * k] (contiguous row ranges
     * balanced by block count, vf_shard_owner_map; row_base(L) = sum over
     * l < L of B_l,y * B_l,z); without it, rank = (j + B_L,y * k) mod count. */
    int32_t shard_rank;
    int32_t shard_count;
    uint8_t *d_row_owner;
    /* embed (bin, face) pair list capacity per level; 0 = 4 F + 65536.  An
     * overflow latches VF_ECAPACITY with the required count in d_status[3]
     * (EmbedEngine re-sizes and reruns). */
    int64_t pair_cap;
    /* cut-link line record capacity (the enumeration's piercing lines);
     * 0 = max(2 F, 2^22).  Lines beyond it are redone by a slower exact
     * kernel (EmbedEngine sizes it from the surface area and re-sizes after
     * its first run); the band list holds max(2^20, line_cap / 16). */
    int64_t line_cap;
} vf_config;

/* ForestGrid as flat device arrays, ids grouped by level:
 * level L occupies ids [level_start[L], level_start[L+1]). */
typedef struct {
    int32_t *d_coords;      /* [cap*4]  i, j, k, level                      */
    int32_t *d_nbr;         /* [cap*27] D3Q27 slot order, slot 0 = self     */
    int32_t *d_nbr_child;   /* [cap*27] first child of neighbour or -1      */
    int32_t *d_child;       /* [cap]    first child id or -1                */
    uint8_t *d_bflags;      /* [cap]    VF_BF_* bits                        */
    uint8_t *d_masks;       /* [cap*64] VF_* cell masks, t = I + 4J + 16K   */
    int32_t *d_level_start; /* [VF_MAX_LEVELS+1] device-resident            */
    int32_t *d_status;      /* [4] latched device errors (0 = ok)           */
    uint64_t *d_solid64;    /* [cap]    bit t set: cell t is SOLID (finalize) */
    int32_t  capacity;
    int32_t  n_levels;      /* host-known number of levels present          */
} vf_grid;

/* one BinLevel */
typedef struct {
    int32_t  level;
    int32_t  mode;          /* 0 = x-rays (1D), 1 = all directions (MD)     */
    int32_t *d_counts;      /* [B_L^3]                                      */
    int32_t *d_offsets;     /* [B_L^3]                                      */
    int32_t *d_face_ids;    /* [face_ids_cap]                               */
    int64_t  face_ids_cap;
    int32_t *d_n_face_ids;  /* [1] device-resident total                    */
    int32_t *d_map;         /* [F] compact_map of kept faces (FilterMap)    */
    int32_t *d_n_map;       /* [1] device-resident |compact_map|            */
} vf_bins;

int         vf_abi_version(void);
/* Per-device context: selects `device`, creates its side
 * streams (bins pipeline, cut-link enumeration) and keeps the caller's
 * ncclComm_t (may be NULL; the library issues no NCCL calls itself -- the
 * multi-GPU flag exchanges are the caller's all-reduces between the sharded
 * stage calls).  Returns NULL on error (vf_last_error).  Without a context
 * the streams are created on first use on the current device. */
void       *vf_ctx_create(int device, void *nccl_comm);
int         vf_ctx_destroy(void *ctx);
int         vf_ctx_device(const void *ctx);
/* NCCL communicator created by the library: rank 0 calls vf_nccl_unique_id
 * (128 bytes), the caller shares the bytes (torch.distributed broadcast) and
 * every rank calls vf_ctx_create_nccl.  NULL on error (vf_last_error). */
int         vf_nccl_unique_id(void *out, int out_bytes);
void       *vf_ctx_create_nccl(int device, int nranks, int rank, const void *unique_id);
const char *vf_last_error(void);
int         vf_device_info(int *sm_count, int *cc_major, int *cc_minor);

/* face records: d_faces[F*12] = v1 v2 v3 (record-major, geometry.py:86-88)
 * followed by the host-computed unit normal (geometry.py:90), 96 B/face */
int vf_pack_faces(const double *d_faces_coord, const double *d_normals,
                  int64_t n_faces, double *d_faces, void *stream);

/* exact FP64 SAT (geometry.py:484-500) on arrays -- test hook */
int vf_sat_batch(const double *d_tri, const double *d_box, int64_t n,
                 uint8_t *d_out, void *stream);

/* --- binning --------------------------------------- */
size_t vf_bins_workspace_size(const vf_config *cfg, int64_t n_faces, int level);
/* compute_ray_indicators (Alg.1) */
int vf_ray_indicators(const vf_config *cfg, const double *d_faces,
                      int64_t n_faces, int level, int mode, uint8_t *d_ind,
                      void *stream);
/* compact_filtered_faces */
size_t vf_compact_workspace_size(int64_t n);
int vf_compact(const uint8_t *d_ind, int64_t n, int32_t *d_map,
               int32_t *d_count, void *d_ws, size_t ws_bytes, void *stream);
/* compute_bin_pairs (Alg.2): pairs in
 * face-major emission order (deterministic); d_map NULL = all faces */
int vf_bin_pairs(const vf_config *cfg, const double *d_faces, int64_t n_faces,
                 const int32_t *d_map, const int32_t *d_n_map, int level,
                 int32_t *d_pair_bin, int32_t *d_pair_face, int64_t pair_cap,
                 int32_t *d_n_pairs, int32_t *d_status, void *d_ws,
                 size_t ws_bytes, void *stream);
/* assemble_bins (steps 3-9 PAPER.md:477-479) */
size_t vf_assemble_workspace_size(int64_t pair_cap, int64_t n_bins);
int vf_bin_assemble(const int32_t *d_pair_bin, const int32_t *d_pair_face,
                    const int32_t *d_n_pairs, int64_t pair_cap, int64_t n_bins,
                    int32_t *d_counts, int32_t *d_offsets, int32_t *d_face_ids,
                    void *d_ws, size_t ws_bytes, void *stream);
/* fused build for one level: indicators -> compact -> pairs -> assemble */
int vf_build_bins(const vf_config *cfg, const double *d_faces, int64_t n_faces,
                  int level, int mode, int use_filter, vf_bins *bins,
                  int32_t *d_status, void *d_ws, size_t ws_bytes, void *stream);

/* --- forest ------------------------------------------ */
int vf_init_forest(const vf_config *cfg, vf_grid *grid, void *stream);
/* adapt, refine-only */
size_t vf_adapt_workspace_size(const vf_grid *grid);
int vf_adapt_refine(const vf_config *cfg, vf_grid *grid, int level,
                    void *d_ws, size_t ws_bytes, void *stream);

/* --- voxelizer --------------------------------------- */
/* partial_surface_voxelize (Alg.3) */
int vf_voxelize_level(const vf_config *cfg, vf_grid *grid, int level,
                      const vf_bins *bins, const double *d_faces, void *stream);
/* propagate_external (Alg.5), dir = +1 / -1; with
 * finalize != 0 the apply epilogue also runs finalize_masks */
size_t vf_propagate_workspace_size(const vf_grid *grid);
int vf_propagate_x(const vf_config *cfg, vf_grid *grid, int level, int dir,
                   int finalize, void *d_ws, size_t ws_bytes, void *stream);
int vf_finalize_level(const vf_config *cfg, vf_grid *grid, int level,
                      void *stream);
/* mark_near_wall_refinement */
size_t vf_mark_workspace_size(const vf_grid *grid);
int vf_mark_level(const vf_config *cfg, vf_grid *grid, int level, void *d_ws,
                  size_t ws_bytes, void *stream);
/* identify_boundary_cells, finest level */
int vf_boundary_cells(const vf_config *cfg, vf_grid *grid, int32_t *d_bcount,
                      void *stream);
/* build_boundary_tables: contraction map + N_b (device) */
size_t vf_tables_workspace_size(const vf_grid *grid);
int vf_link_tables(const vf_config *cfg, vf_grid *grid, const int32_t *d_bcount,
                   int32_t *d_cmap, int32_t *d_n_b, void *d_ws, size_t ws_bytes,
                   void *stream);
/* compute_link_lengths: face-parallel, exact min via
 * atomicMin on the IEEE bits; d_lengths[n_b*27*64] must hold -1.0f.
 * d_map/d_n_map: optional filtered face list (NULL = all faces). */
size_t vf_link_workspace_size(const vf_config *cfg, const vf_grid *grid);
int vf_link_lengths(const vf_config *cfg, vf_grid *grid, const int32_t *d_cmap,
                    const double *d_faces, int64_t n_faces,
                    const int32_t *d_map, const int32_t *d_n_map,
                    float *d_lengths, void *d_ws, size_t ws_bytes, void *stream);

/* --- embed_geometry driver ----------------------------
 * Phase 1 (no host sync): init_forest + per level bins/voxelize/propagate/
 * finalize/mark/adapt + finest boundary cells + tables.  Writes the
 * contraction map into d_cmap[capacity] and N_b into d_n_b.
 * Phase 2: LUT initialisation (-1) for the device-resident N_b and link
 * lengths into d_lengths (capacity lengths_cap boundary blocks).  Stage
 * events (optional, 64 cudaEvent_t) bracket the phase-1 stages. */
size_t vf_embed_workspace_size(const vf_config *cfg, int64_t n_faces,
                               int32_t capacity);
int vf_embed_phase1(const vf_config *cfg, const double *d_faces,
                    int64_t n_faces, int use_filter, vf_grid *grid,
                    int32_t *d_cmap, int32_t *d_n_b, void *d_ws,
                    size_t ws_bytes, void *stream, void **events);
int vf_embed_phase2(const vf_config *cfg, const double *d_faces,
                    int64_t n_faces, vf_grid *grid, const int32_t *d_cmap,
                    const int32_t *d_n_b, float *d_lengths, int64_t lengths_cap,
                    void *d_ws, size_t ws_bytes, void *stream,
                    void **link_events /* 2 or NULL */);
/* Both phases captured as one CUDA graph (no host sync inside: the LUT is
 * filled for the device-resident N_b; N_b > lengths_cap latches
 * VF_ECAPACITY).  `stream` must not be the legacy default stream. */
int vf_embed_graph_create(const vf_config *cfg, const double *d_faces,
                          int64_t n_faces, int use_filter, vf_grid *grid,
                          int32_t *d_cmap, int32_t *d_n_b, float *d_lengths,
                          int64_t lengths_cap, void *d_ws, size_t ws_bytes,
                          void *stream, void **graph_exec);
int vf_graph_launch(void *graph_exec, void *stream);
void vf_graph_destroy(void *graph_exec);
/* wait for the library's per-device side streams (phase 1 launches the
 * grid-independent cut-link enumeration there; phase 2 joins it).  Call after
 * a phase 1 that is not followed by phase 2 before releasing its workspace. */
int vf_side_sync(void);
/* End-to-end (serving) formats.  vf_pack_indexed: the engine's 96-B face
 * records from an indexed mesh -- the reference TriangleMesh's vertices (V,3)
 * f64 and faces_indexed (F,3) (here int32) -- with the unit normals computed
 * as TriangleMesh._face_normals does (geometry.py:114-124, np.cross / norm,
 * bit-identical); an out-of-range index or a zero normal latches VF_EMESH in
 * d_status.  vf_lut_sparse: the cut links of lengths[N_b][27][64] (N_b read
 * from d_n_b) as (flat index, q) pairs in index order -- the index is the
 * unsigned 32-bit (slot * 27 + q) * 64 + t stored in int32 --; *d_count = the
 * number of links (only the first `cap` are written). */
int vf_pack_indexed(const double *verts, int64_t V, const int32_t *faces_idx, int64_t F, double *out,
                    int32_t *d_status, void *stream);
size_t vf_lut_sparse_workspace_size(int64_t lengths_cap);
int vf_lut_sparse(const float *lengths, int64_t lengths_cap, const int32_t *d_n_b, int32_t *idx, float *val,
                  int64_t cap, int32_t *d_count, void *ws, size_t ws_bytes, void *stream);
/* number of kernels this library has launched in the process (bench hook) */
int64_t vf_launch_count(void);
/* Per-kernel timer (bench / profiling hook).  vf_ktimer_start: the embed
 * calls that follow on `stream` run every kernel on that stream in order (no
 * side streams) behind a spin kernel of `gate_us` microseconds, and an event
 * is recorded after every launch and memset.  vf_ktimer_stop synchronises and
 * writes "name<TAB>launches<TAB>total ms\n" lines (first-appearance order)
 * into buf; returns the byte count (negative status on a CUDA error). */
int vf_ktimer_start(void *stream, double gate_us);
int vf_ktimer_stop(char *buf, int buflen);

/* Counters of the last embed's cut-link pass on this workspace (synchronous):
 * out[7] = {piercing lines recorded, line capacity, faces whose lines
 * overflowed (redone by the direct kernel), band candidates, band capacity,
 * faces enumerated by the large-face kernel, lattice lines classified by the
 * enumeration (FP32 intersection tests)}. */
int vf_embed_link_stats(const vf_config *cfg, int64_t F, int32_t capacity, void *ws, size_t ws_bytes,
                        int64_t *out);
/* multi-GPU exchange helper: zero the level-L entries of blocks this rank
 * does not own (block flags, solid64 and, if given, d_bcount) so that one
 * all-reduce (MAX for flags, SUM for solid64/bcount) publishes the owners'
 * values to every rank */
int vf_shard_zero_unowned(const vf_config *cfg, vf_grid *grid, int level,
                          int32_t *d_bcount, void *stream);
/* ---- block-sharded multi-GPU embed (one process per GPU; the caller runs
 * the NCCL exchanges between these calls, see parallel.py).  All use the
 * embed workspace (vf_embed_workspace_size) and cfg->shard_rank/count/
 * d_row_owner.
 * size of cfg->d_row_owner (bytes): one owner byte per block row per level */
size_t vf_shard_owner_bytes(const vf_config *cfg);
/* owner map of level L from the (replicated) level-L blocks: contiguous row
 * ranges with equal block counts, identical on every rank */
int vf_shard_owner_map(const vf_config *cfg, vf_grid *grid, int level, void *d_ws,
                       size_t ws_bytes, void *stream);
/* level L on the owned rows: bins (Alg. 1-2, owned rows/bins), voxelize,
 * Alg. 5 (+x, -x) + finalize, then zero the level's flags / solid64 of
 * unowned blocks for the owner-zeroed all-reduce */
int vf_shard_level(const vf_config *cfg, const double *d_faces, int64_t n_faces,
                   int use_filter, vf_grid *grid, int level, void *d_ws, size_t ws_bytes,
                   void *stream);
/* replicated refinement of level L (mark + adapt) and the owner map of L+1 */
int vf_shard_refine(const vf_config *cfg, vf_grid *grid, int level, void *d_ws,
                    size_t ws_bytes, void *stream);
/* finest level: boundary cells of owned blocks (counts -> d_bcount, zeroed
 * for unowned blocks) */
int vf_shard_boundary(const vf_config *cfg, vf_grid *grid, int32_t *d_bcount, void *stream);
/* native sharded embed through the tables: every level above with the
 * block-flag all-reduce (MAX) on ctx's NCCL communicator, then the finest
 * level's SOLID-mask and boundary-count all-reduces and the replicated
 * tables; stream-ordered, no host sync (graph-capturable).  ctx from
 * vf_ctx_create_nccl or vf_ctx_create with the caller's ncclComm_t. */
int vf_shard_embed_phase1(void *ctx, const vf_config *cfg, const double *d_faces, int64_t n_faces,
                          int use_filter, vf_grid *grid, int32_t *d_bcount, int32_t *d_cmap,
                          int32_t *d_n_b, void *d_ws, size_t ws_bytes, void *stream);
/* cut-link LUT slots of the owned blocks: LUT init (-1), faces near owned
 * rows, k_links on them (the LUT stays distributed) */
int vf_shard_links(const vf_config *cfg, const double *d_faces, int64_t n_faces,
                   vf_grid *grid, const int32_t *d_cmap, const int32_t *d_n_b,
                   float *d_lengths, int64_t lengths_cap, void *d_ws, size_t ws_bytes,
                   void *stream);
/* ---- LUT consumer: D3Q27 BGK collide/stream of
 * one level with SBB / interpolated bounce-back walls from the LinkTable
 * (SPEC.md:398-411).  State = post-collision populations f[27][(e-s)*64]
 * (f32, SoA) over the level's block ids [s, e). */
typedef struct {
    double tau;       /* BGK relaxation time of the level (> 1/2)          */
    double u_in[3];   /* inlet velocity (lattice units) at the x = 0 face  */
    int32_t ibb;      /* 1 = Bouzidi linear IBB from the LUT, 0 = SBB      */
    int32_t open_x;   /* 1 = inlet (x = 0) / outlet (x = l_x) faces, 0 = SBB */
} vf_flow;
int vf_lbm_init(const vf_grid *grid, int32_t s, int32_t e, double rho, const double *u,
                float *d_f, void *stream);
/* one step: d_fout = collide(stream(d_fin)); the wall-link momentum exchange
 * is ADDED to d_force[3] (lattice units) when d_force is not NULL, summed in
 * block order (deterministic).  d_scratch: 7 (e - s) + 4 int32 (the list of
 * blocks with a non-simple cell -- SOLID / GHOST / next to a wall, a missing
 * block or the domain boundary -- then 3 doubles of per-block force partials) */
int vf_lbm_step(const vf_config *cfg, const vf_grid *grid, int level, int32_t s, int32_t e,
                const int32_t *d_cmap, const float *d_lengths, const float *d_fin,
                float *d_fout, const vf_flow *flow, double *d_force, int32_t *d_scratch,
                void *stream);
/* ---- interface exchange between levels L and L+1 (SPEC.md:417-424,
 * SURVEY.md §8(f) next #3).  Block ranges: fine [sf, ef) at L+1, coarse
 * [sc, ec) at L; states are the levels' post-collision f[27][...] arrays.
 * vf_lbm_parents: d_parent[b] = parent block of every child (-1 elsewhere)
 * over ids [0, n_blocks).
 * vf_lbm_fill_ghosts: fine GHOST cells <- tensor-product interpolation
 * ([sf, ef) a whole level >= 1: groups of 8 siblings, else VF_EARG)
 * (order 3 cubic / 1 linear / 0 copy, falling back when a stencil cell is
 * outside the level or SOLID) of (1 - theta) fc_old + theta fc_new, then
 * f = feq + alpha (f - feq) (alpha = 1: no rescale).
 * vf_lbm_restrict: coarse cells of refined blocks (not SOLID / INTERFACE /
 * GHOST, no GHOST child) <- mean of their non-SOLID children, rescaled by
 * beta ([sf, ef) whole sibling groups as for the fill; d_parent as there). */
int vf_lbm_parents(const vf_grid *grid, int32_t n_blocks, int32_t *d_parent, void *stream);
int vf_lbm_fill_ghosts(const vf_grid *grid, int32_t sf, int32_t ef, int32_t sc, int32_t ec,
                       const int32_t *d_parent, const float *d_fc_old, const float *d_fc_new,
                       double theta, double alpha, int order, float *d_ff, void *stream);
int vf_lbm_restrict(const vf_grid *grid, int32_t sc, int32_t ec, int32_t sf, int32_t ef,
                    const int32_t *d_parent, const float *d_ff, double beta, float *d_fc, void *stream);
/* copy the grid's latched device status to the host (synchronizes) */
int vf_check_status(const vf_grid *grid, void *stream);
/* test hook: capacity of the link-length band list (candidates the FP32
 * classifier leaves to the exact SAT; default 1<<20).  A smaller value forces
 * the overflow fallback pass; results are identical.  Returns the old value;
 * n < 0 only queries. */
int64_t vf_set_link_band_cap(int64_t n);

/* Measurement hook: 1 = run the cut-link line enumeration serially on the
 * caller's stream after the tables (its events then time the kernel alone),
 * 0 = overlapped on the side stream (default; results identical).  Returns
 * the old value; on < 0 only queries.  Affects graphs created afterwards. */
int vf_set_serial_links(int on);

/* Tuning / test hook: faces whose bounding box spans at most e cells are
 * enumerated thread per face (k_links_small), larger ones by the
 * warp-flattened kernel (default 1.5; results identical for any e; e < 0
 * sends every face to the large-face kernel).  Returns the old value; NaN
 * only queries. */
float vf_set_link_small_ext(float e);

/* Test hook: 1 = Alg. 5 rows through the chunked kernel at every level,
 * 0 = the shared-memory staged kernel for rows of <= 128 blocks (default;
 * results identical).  Returns the old value; on < 0 only queries. */

#ifdef __cplusplus
}
#endif
#endif
