/*
 * actmap_b200.h -- C ABI of the B200-native oMAP hot path.
 *
 * This is the drop-in boundary under the reference's actmap:: planner API
 * (/root/reference/proj/core/include/actmap/).  Plain pointers and sizes,
 * status codes instead of exceptions, caller-owned host buffers,
 * context-owned device buffers; a context is externally synchronised (one
 * host thread at a time).  Every entry point names the reference interface
 * it serves.  The C++ API (the include/actmap/ headers, same signatures as the
 * reference headers) is implemented on top of these calls, and INTEGRATION.md
 * shows the ctypes / C++ bindings.
 *
 * Status -> reference exception (errors.hpp:10-44):
 *   AM_EINVAL      -> actmap::InvalidInputError  (CLI exit 1)
 *   AM_EUNCOVERED  -> actmap::UncoveredTargetError (CLI exit 2; per target in batch calls)
 *   AM_ECUDA/AM_EOOM/AM_ENCCL/AM_EINTERNAL -> actmap::Error
 */
#ifndef ACTMAP_B200_H
#define ACTMAP_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define AM_ABI_VERSION 1

typedef enum am_status {
  AM_OK = 0,
  AM_EINVAL = 1,
  AM_EUNCOVERED = 2,
  AM_ECUDA = 3,
  AM_EOOM = 4,
  AM_ENCCL = 5,
  AM_EINTERNAL = 6
} am_status;

/* propagate.hpp:45-49 (AutoStop) plus the fixed-L case of report.hpp:75. */
enum { AM_STOP_FILLED = 0, AM_STOP_STALLED = 1, AM_STOP_CAP = 2, AM_STOP_FIXED = 3 };
/* propagate.hpp:22 */
enum { AM_MODE_BATCHED = 0, AM_MODE_ITERATIVE = 1 };
/* report.hpp:15 */
enum { AM_METHOD_SIMPLE = 0, AM_METHOD_EUCLIDEAN = 1 };

typedef struct am_ctx am_ctx;
typedef struct am_grid am_grid;

#define AM_CTX_TIMING 1u /* time every stencil block launch with CUDA events */
#define AM_CTX_DENSE 2u  /* disable exact active-tile skipping: every block sweeps the whole grid */

typedef struct am_ctx_opts {
  int32_t device; /* CUDA ordinal */
  uint32_t flags; /* AM_CTX_* */
} am_ctx_opts;

typedef struct am_prop_result {
  uint32_t layers_used;     /* AutoResult::layers_used (propagate.hpp:53) */
  uint32_t cause;           /* AM_STOP_* (AutoResult::cause, propagate.hpp:54) */
  uint32_t layers_computed; /* layers actually run on the device (>= layers_used; overshoot rolled back exactly) */
  uint32_t cell_bits;       /* final device cell width (16 or 32) */
  uint64_t block_launches;  /* temporally blocked stencil launches */
  uint64_t layer_launches;  /* single-layer stencil launches */
  double stencil_ms;        /* summed CUDA-event time of the block launches (AM_CTX_TIMING) */
  uint64_t tiles_processed; /* tile-blocks computed with active-tile skipping (0 in dense mode) */
  uint64_t tiles_total;     /* tiles per grid x blocks: the dense-equivalent tile-blocks */
  uint64_t cells_executed;  /* cell-updates the blocked launches computed (processed tiles x tile cells x layers) */
  uint32_t engine;          /* AM_ENGINE_*: which blocked kernel ran the bulk of the layers */
  uint32_t block_layers;    /* layers per blocked launch of that kernel */
} am_prop_result;

/* am_prop_result.engine */
enum { AM_ENGINE_DENSE = 0, AM_ENGINE_TILES = 1, AM_ENGINE_BITS = 2, AM_ENGINE_BATCH = 3 };

typedef struct am_grid_info {
  uint32_t width, height, pitch, rows, bands, segments, seg_len, halo;
  uint32_t cell_bits, layers_used, layers_computed;
  uint32_t tile_rows, tile_cols, tiles; /* active-tile geometry (tiles = 0 for slab grids) */
} am_grid_info;

typedef struct am_stats {
  uint64_t kernel_launches; /* every kernel this context has launched */
  uint64_t pool_reserved;   /* device bytes held by the context's memory pool */
  uint64_t pool_used;       /* of which in use by live grids / scratch */
  uint64_t h2d_bytes;       /* host-to-device bytes this context has copied (occupancy, sources, targets) */
} am_stats;

/* ---- context ---------------------------------------------------------- */
am_status am_ctx_create(const am_ctx_opts *opts, am_ctx **out);
void am_ctx_destroy(am_ctx *ctx);
const char *am_last_error(const am_ctx *ctx);
am_status am_ctx_stats(const am_ctx *ctx, am_stats *out);
am_status am_ctx_synchronize(am_ctx *ctx);
/* Device memory of destroyed grids stays cached in the context's stream-
 * ordered pool for the next grid (no cudaMalloc/cudaFree per solve); this
 * returns the unused part to the driver. */
am_status am_ctx_trim(am_ctx *ctx);
/* The cudaStream_t every kernel of this context is launched on (so callers
 * can bracket work with CUDA events on the launching stream). */
am_status am_ctx_get_stream(const am_ctx *ctx, void **stream);
/* Pinned, device-mapped host memory on the context's device.  Host buffers of
 * this kind are written by the kernels directly (am_trace_paths streams the
 * points into them while the paths are walked; am_grid_create reads them with
 * the copy engine); any other host pointer is staged.  No reference
 * counterpart: the C++ API (actmap_api.cpp) keeps its trace buffers here. */
am_status am_host_alloc(am_ctx *ctx, size_t bytes, void **out);
am_status am_host_free(am_ctx *ctx, void *p);

/* ---- grid + sources (GridMap grid.hpp:18-57, SourceSet grid.hpp:80-90) --
 * occupancy: width*height bytes, row-major, nonzero = obstacle.
 * src_rc: n_src (row, col) pairs; each in bounds and free, n_src >= 1
 * (duplicates collapse).  *_device variants take device pointers (inputs
 * already resident in HBM). */
am_status am_grid_create(am_ctx *ctx, uint32_t width, uint32_t height, const uint8_t *occupancy,
                         const uint32_t *src_rc, uint64_t n_src, am_grid **out);
am_status am_grid_create_device(am_ctx *ctx, uint32_t width, uint32_t height, const uint8_t *d_occupancy,
                                const uint32_t *d_src_rc, uint64_t n_src, am_grid **out);
am_status am_grid_destroy(am_ctx *ctx, am_grid *grid);
/* A new grid with the same occupancy and SourceSet, built on the device from
 * `grid`'s resident copies (no host data; `grid` may be destroyed after).
 * New surface: it keeps the value semantics of maps a planner returned
 * (ActivityMap is returned by value, activity.hpp:17-18) without holding
 * on to the caller's GridMap. */
am_status am_grid_clone(am_ctx *ctx, const am_grid *grid, am_grid **out);
am_status am_grid_get_info(const am_grid *grid, am_grid_info *out);

/* ---- propagation (propagate.hpp:40-61) ---------------------------------
 * layers >= 1: fixed L (propagate); layers == 0: auto mode with auto_cap
 * (propagate_auto).  mode: AM_MODE_BATCHED (temporally blocked) or
 * AM_MODE_ITERATIVE (one launch + host-visible boundary per layer); outputs
 * are bit-identical.  The map stays resident on the device. */
am_status am_propagate(am_ctx *ctx, am_grid *grid, uint32_t layers, uint32_t auto_cap, uint32_t mode,
                       am_prop_result *res);

/* ActivityMap::values() (activity.hpp:40): dense row-major uint32 W*H. */
am_status am_activity_download(am_ctx *ctx, am_grid *grid, uint32_t *dense_host);
am_status am_activity_download_device(am_ctx *ctx, am_grid *grid, uint32_t *dense_device);
/* Replace the grid's map by a caller-supplied dense map (reconstruct on an
 * ActivityMap that did not come from am_propagate; reconstruct.hpp:38,45). */
am_status am_activity_upload(am_ctx *ctx, am_grid *grid, const uint32_t *dense_host, uint32_t layers_applied);

/* ---- path extraction (reconstruct.hpp:34-47), batched over targets ------
 * Step 1: am_path_counts -> offsets[0..n] (exclusive scan; offsets[n] =
 * total points) and per-target status (AM_OK / AM_EINVAL / AM_EUNCOVERED).
 * Step 2: am_trace_paths writes target->source points (row, col pairs) at
 * pts_rc[2*offsets[i] ..].  method: AM_METHOD_*; seed: simple-method
 * tie-break seed (pin P2).  Euclidean paths are returned straightened
 * (strict corner rule); for maps produced by am_propagate straightening is
 * provably the identity and is skipped. */
am_status am_path_counts(am_ctx *ctx, am_grid *grid, const uint32_t *tgt_rc, uint64_t n, uint32_t method,
                         uint64_t seed, uint64_t *offsets, int32_t *status);
am_status am_trace_paths(am_ctx *ctx, am_grid *grid, const uint32_t *tgt_rc, uint64_t n, uint32_t method,
                         uint64_t seed, const uint64_t *offsets, uint32_t *pts_rc, uint64_t pts_capacity,
                         int32_t *status);
/* Device-resident variant: targets, offsets (n+1), points and status are
 * device pointers; counts, scan and trace run back to back on the stream
 * with no host round trip.  A target whose points would end past
 * pts_capacity gets status AM_EINVAL and nothing is written for it. */
am_status am_trace_paths_device(am_ctx *ctx, am_grid *grid, const uint32_t *d_tgt_rc, uint64_t n,
                                uint32_t method, uint64_t seed, uint64_t *d_offsets, uint32_t *d_pts_rc,
                                uint64_t pts_capacity, int32_t *d_status);

/* ---- single-shot entry points over host buffers ------------------------ */
/* propagate_layer (propagate.hpp:37-38): one layer from an arbitrary map. */
am_status am_propagate_layer(am_ctx *ctx, uint32_t width, uint32_t height, const uint8_t *occupancy,
                             const uint32_t *src_rc, uint64_t n_src, const uint32_t *in, uint32_t *out);
/* propagate_reference (propagate.hpp:67-68): literal INT32_MIN sentinel kernel. */
am_status am_propagate_reference(am_ctx *ctx, uint32_t width, uint32_t height, const uint8_t *occupancy,
                                 const uint32_t *src_rc, uint64_t n_src, uint32_t layers, uint32_t *out);

/* ---- benchmark hook (tools/tile_probe.py) ------------------------------
 * Times the active-tile kernel alone: `items` work items (pairs of tiles,
 * chosen `stride` tiles apart, all at layer 0) launched `reps` times on the
 * grid's layer-0 map; writes the mean launch time.  Leaves the grid without
 * a map (propagate again before reading it). */
am_status am_bench_tile_kernel(am_ctx *ctx, am_grid *grid, uint32_t items, uint32_t stride, uint32_t reps,
                               float *ms_per_launch);

/* ---- multi-GPU row slabs ---------------------------------
 * A slab grid owns rows [row0, row1) of a width x height grid; occupancy is
 * the FULL grid (host), sources use global coordinates.  Slabs keep K=8
 * halo rows refreshed before every launch.
 *
 * One process per GPU: am_comm_unique_id on one rank, share the 128 bytes,
 * am_comm_init on every rank, am_comm_slab_rows for this rank's rows, then
 * am_propagate on the slab grid (NCCL halo send/recv + flag all-reduce) and
 * am_comm_gather into a full-size grid (am_grid_create) to trace paths.
 *
 * In-process (one device): am_slabs_propagate drives n consecutive slabs
 * created on the same context; am_slabs_gather assembles the full map. */
am_status am_grid_create_slab(am_ctx *ctx, uint32_t width, uint32_t height, uint32_t row0, uint32_t row1,
                              const uint8_t *occupancy_full, const uint32_t *src_rc, uint64_t n_src, am_grid **out);
am_status am_slabs_propagate(am_ctx *ctx, am_grid **slabs, uint32_t n, uint32_t layers, uint32_t auto_cap,
                             uint32_t mode, am_prop_result *res);
am_status am_slabs_gather(am_ctx *ctx, am_grid **slabs, uint32_t n, am_grid *full);
am_status am_comm_unique_id(uint8_t *id_out /* 128 bytes */);
am_status am_comm_init(am_ctx *ctx, uint32_t nranks, uint32_t rank, const uint8_t *id /* 128 bytes */);
am_status am_comm_slab_rows(const am_ctx *ctx, uint32_t height, uint32_t *row0, uint32_t *row1);
am_status am_comm_gather(am_ctx *ctx, am_grid *slab, am_grid *full);
/* rows [row0, row1) of slab `rank` of `nranks` over `height` rows (the cut
 * am_comm_slab_rows uses; no communicator needed).  New surface (SURVEY.md
 * §8e): the reference's only parallelism is the `threads` knob of
 * propagate (propagate.hpp:30-31), with results invariant in it. */
am_status am_slab_rows(uint32_t height, uint32_t nranks, uint32_t rank, uint32_t *row0, uint32_t *row1);

/* ---- peer-memory slab transport (no NCCL call on the per-block path) -----
 * One process per GPU (or several on one GPU).  Each rank's slab exports a
 * blob (CUDA IPC handles of its halo inbox, its publish buffer and its block
 * events); the caller shares the blobs (any host channel, e.g.
 * torch.distributed all_gather_object) and connects.  Per block, the
 * boundary kernel stores the slab's first / last K rows straight into the
 * neighbours' inboxes through the mapped peer pointers (NVLink / NVSwitch
 * P2P stores across GPUs), records an IPC event, and the neighbours' streams
 * wait on it (stream-ordered: no kernel spins on another rank).  The
 * fixed-point words ride along as in the NCCL transport.  am_propagate on a
 * connected slab uses this transport; am_peer_gather assembles the full map
 * from the peers' published slabs with peer-to-peer copies. */
#define AM_PEER_BLOB_BYTES 1024
am_status am_peer_export(am_ctx *ctx, am_grid *slab, uint8_t *blob /* AM_PEER_BLOB_BYTES */);
am_status am_peer_connect(am_ctx *ctx, am_grid *slab, uint32_t nranks, uint32_t rank,
                          const uint8_t *blobs /* nranks x AM_PEER_BLOB_BYTES, rank order */);
am_status am_peer_gather(am_ctx *ctx, am_grid *slab, am_grid *full);
/* am_trace_paths_device on the map distributed over the connected slabs: every
 * rank publishes its rows, then the walkers read across slab edges through
 * the peer-mapped publish buffers (no full-map gather).  Any rank may trace
 * any target (grid coordinates); every rank must call it (the publish is a
 * rendezvous), with n = 0 if it has no targets. */
am_status am_peer_trace_paths_device(am_ctx *ctx, am_grid *slab, const uint32_t *d_tgt_rc, uint64_t n,
                                     uint32_t method, uint64_t seed, uint64_t *d_offsets, uint32_t *d_pts_rc,
                                     uint64_t pts_capacity, int32_t *d_status);

/* ---- small-grid batch (BASELINE.json config 5) ---------------------------
 * n independent width x height mazes solved in one device run: the
 * reference's propagate / propagate_auto / reconstruct_* applied to every
 * maze, results per maze.  occupancy: n*height*width bytes (maze-major);
 * sources of maze i: src_rc[2*src_off[i] .. 2*src_off[i+1]) (maze-local
 * (row, col)); targets: (maze, row, col) triples; path points come back in
 * maze-local coordinates. */
typedef struct am_batch am_batch;
am_status am_batch_create(am_ctx *ctx, uint32_t n_mazes, uint32_t width, uint32_t height, const uint8_t *occupancy,
                          const uint64_t *src_off, const uint32_t *src_rc, am_batch **out);
am_status am_batch_destroy(am_ctx *ctx, am_batch *batch);
am_status am_batch_propagate(am_ctx *ctx, am_batch *batch, uint32_t layers, uint32_t auto_cap,
                             uint32_t *layers_used /* n */, uint32_t *cause /* n */, am_prop_result *global);
am_status am_batch_download(am_ctx *ctx, am_batch *batch, uint32_t *maps /* n*height*width */);
am_status am_batch_path_counts(am_ctx *ctx, am_batch *batch, const uint32_t *tgt_mrc, uint64_t n, uint32_t method,
                               uint64_t seed, uint64_t *offsets, int32_t *status);
am_status am_batch_trace_paths(am_ctx *ctx, am_batch *batch, const uint32_t *tgt_mrc, uint64_t n, uint32_t method,
                               uint64_t seed, const uint64_t *offsets, uint32_t *pts_rc, uint64_t pts_capacity,
                               int32_t *status);

/* ---- map / scene text I/O (mapio.hpp:19-38) ------------
 * The text goes to the device once; newline scan, row validation,
 * character classes and the source / target lists are computed there (the
 * occupancy never exists on the host unless downloaded).  Parse failures
 * return AM_EINVAL and fill am_parse_info: error_line / error_column
 * (1-based, 0 when the error has no position) map to actmap::ParseError,
 * otherwise to InvalidInputError (errors.hpp:23-38). */
enum { AM_FORMAT_MOVINGAI = 0, AM_FORMAT_ASCII_SCENE = 1 };
typedef struct am_parse_info {
  uint32_t width, height;
  uint64_t n_sources, n_targets, obstacles;
  uint64_t error_line, error_column;
  char error[160];
} am_parse_info;
typedef struct am_scene am_scene;
/* Moving AI header only (host, no device): width/height and the byte offset
 * of the first map row.  parse_movingai's header rules (mapio.hpp:19-22). */
am_status am_movingai_header(const char *text, uint64_t len, am_parse_info *info, uint64_t *body_offset);
/* parse_movingai (mapio.hpp:23) / parse_ascii_scene (mapio.hpp:30) into a
 * device-resident scene: occupancy, and for ASCII scenes the 'S' sources and
 * 'T' targets in row-major order. */
am_status am_scene_parse(am_ctx *ctx, const char *text, uint64_t len, uint32_t format, am_scene **out,
                         am_parse_info *info);
am_status am_scene_destroy(am_ctx *ctx, am_scene *scene);
/* any pointer may be NULL; sizes: W*H bytes and 2*n u32 (see am_parse_info) */
am_status am_scene_download(am_ctx *ctx, const am_scene *scene, uint8_t *occupancy, uint32_t *src_rc,
                            uint32_t *tgt_rc);
/* build_grid + SourceSet straight from a parsed scene (no host occupancy);
 * src_rc NULL = the scene's own sources, else n_src host (row, col) pairs
 * (sources given by the caller override the file). */
am_status am_grid_create_scene(am_ctx *ctx, const am_scene *scene, const uint32_t *src_rc, uint64_t n_src,
                               am_grid **out);
/* emit_movingai (mapio.hpp:26) / emit_ascii_scene (mapio.hpp:32): the text of
 * a grid ('.'/'@' or '.'/'#' plus 'S'/'T').  out NULL: *length only. */
am_status am_emit_text(am_ctx *ctx, uint32_t format, uint32_t width, uint32_t height, const uint8_t *occupancy,
                       const uint32_t *src_rc, uint64_t n_src, const uint32_t *tgt_rc, uint64_t n_tgt, char *out,
                       uint64_t capacity, uint64_t *length);
/* export_pgm (mapio.hpp:35-38): binary P5 of the grid's map (device-resident)
 * or of a host map; maxval 255, or 65535 when the maximum exceeds 255.  out
 * NULL: *length only. */
am_status am_activity_export_pgm(am_ctx *ctx, am_grid *grid, uint8_t *out, uint64_t capacity, uint64_t *length);
am_status am_export_pgm(am_ctx *ctx, uint32_t width, uint32_t height, const uint32_t *values, uint8_t *out,
                        uint64_t capacity, uint64_t *length);

/* ---- host helpers of the planner API (no device work) ------------------ */
/* random_maze / comb_maze (grid.hpp:65-76) into a caller buffer of W*H bytes. */
am_status am_random_maze(uint32_t width, uint32_t height, double density, uint64_t seed, uint8_t *occupancy);
am_status am_comb_maze(uint32_t width, uint32_t height, uint8_t *occupancy);
/* benchmark workloads: C2 perfect maze, C3 city blocks (new, not in the reference) */
am_status am_kruskal_maze(uint32_t width, uint32_t height, uint64_t seed, uint8_t *occupancy);
am_status am_city_grid(uint32_t width, uint32_t height, uint64_t seed, uint8_t *occupancy);
/* straighten (reconstruct.hpp:49-58); occupancy may be NULL for the
 * geometric variant; rule 0 = strict, 1 = permissive.  out may alias pts. */
am_status am_straighten(const uint32_t *pts_rc, uint64_t n, const uint8_t *occupancy, uint32_t width,
                        uint32_t height, uint32_t rule, uint32_t *out_rc, uint64_t *n_out);
/* path_metrics (reconstruct.hpp:26-32). */
am_status am_path_metrics(const uint32_t *pts_rc, uint64_t n, uint64_t *steps, double *euclidean_length);

#ifdef __cplusplus
}
#endif
#endif
