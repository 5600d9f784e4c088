/*
 * actmap_oracle.h -- CPU restatement of the oMAP reference algorithm.
 *
 * TEST INFRASTRUCTURE ONLY.  This library is the parity checker and the CPU
 * baseline.  Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference legs may load it.  The product library
 * (paper_2004_00540_b200/libactmap_b200.so) never links or calls it.
 *
 * Parity status: the reference ships declarations only (no function bodies,
 * see SURVEY.md §0), so there is no reference binary to run.  The oracle is
 * pinned by (a) every worked example in /root/reference/SPEC.md (golden
 * vectors in tests/golden/spec_kats.json, checked in tests/test_oracle.py),
 * (b) the closed-form activity law of activity.hpp:12-14 / SPEC.md:98,153
 * checked against an independent breadth-first search, and (c) the literal
 * sentinel formulation (propagate.hpp:63-68) checked elementwise against the
 * mask formulation.  Path point sequences follow the builder pins P1/P2/P4
 * (SURVEY.md Appendix); the simple-method sequence is defined by pin P2
 * because the reference leaves its generator unspecified.
 *
 * Layouts follow the reference exactly: occupancy is row-major uint8 with
 * nonzero = obstacle (grid.hpp:20), activity is row-major uint32
 * (activity.hpp:51), coordinates are (row, col) pairs (coord.hpp:13-18).
 */
#ifndef ACTMAP_ORACLE_H
#define ACTMAP_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum {
  OR_OK = 0,
  OR_EINVAL = 1,      /* actmap::InvalidInputError (errors.hpp:17) */
  OR_EUNCOVERED = 2,  /* actmap::UncoveredTargetError (errors.hpp:41) */
  OR_EINTERNAL = 6    /* map violates the ascent invariant */
};

#define OR_UNREACH 0xFFFFFFFFu          /* oracle.hpp:14 kUnreachableHops */
#define OR_MAX_LAYERS 2147483646u       /* propagate.hpp:15-16 kMaxLayers */
#define OR_MAX_DIM 65535u               /* grid.hpp:14 kMaxGridDim */

enum { OR_STOP_FILLED = 0, OR_STOP_STALLED = 1, OR_STOP_CAP = 2 }; /* propagate.hpp:45-49 */
enum { OR_CORNER_STRICT = 0, OR_CORNER_PERMISSIVE = 1 };           /* reconstruct.hpp:14 */
enum { OR_MODE_BATCHED = 0, OR_MODE_ITERATIVE = 1 };               /* propagate.hpp:22 */

/* ---- randomness (pin P2 / generator pins) ---- */
uint64_t or_splitmix64(uint64_t *state);
/* floor(u * n / 2^64): unbiased-enough bounded draw, platform exact. */
uint64_t or_bounded(uint64_t u, uint64_t n);

/* ---- generators (grid.hpp:62-76) ---- */
int or_random_maze(uint32_t w, uint32_t h, double density, uint64_t seed, uint8_t *occ);
int or_comb_maze(uint32_t w, uint32_t h, uint8_t *occ);
int or_kruskal_maze(uint32_t w, uint32_t h, uint64_t seed, uint8_t *occ);
int or_city_grid(uint32_t w, uint32_t h, uint64_t seed, uint8_t *occ);
/* n distinct free cells, none of them flagged in `exclude` (nullable, 1 B/cell). */
int or_sample_free_cells(uint32_t w, uint32_t h, const uint8_t *occ, uint64_t n,
                         uint64_t seed, const uint8_t *exclude, uint32_t *rc_out);

/* ---- SourceSet (grid.hpp:80-90): validates and rasterises to a 0/1 mask ---- */
int or_source_mask(uint32_t w, uint32_t h, const uint8_t *occ, const uint32_t *src_rc,
                   uint64_t n_src, uint8_t *srcmask);

/* ---- propagation (propagate.hpp:34-79) ---- */
int or_initial(uint32_t w, uint32_t h, const uint8_t *occ, const uint8_t *srcmask, uint32_t *out);
int or_propagate_layer(uint32_t w, uint32_t h, const uint8_t *occ, const uint8_t *srcmask,
                       const uint32_t *in, uint32_t *out, int threads);
int or_propagate(uint32_t w, uint32_t h, const uint8_t *occ, const uint8_t *srcmask,
                 uint32_t layers, int mode, int threads, uint32_t *out);
int or_propagate_auto(uint32_t w, uint32_t h, const uint8_t *occ, const uint8_t *srcmask,
                      uint32_t auto_cap, int threads, uint32_t *out,
                      uint32_t *layers_used, int *cause);
int or_propagate_reference(uint32_t w, uint32_t h, const uint8_t *occ, const uint8_t *srcmask,
                           uint32_t layers, uint32_t *out);
void or_layer_bound(uint32_t w, uint32_t h, uint64_t *worst, uint32_t *lo, uint32_t *hi);
uint64_t or_zero_free_cells(uint32_t w, uint32_t h, const uint8_t *occ, const uint32_t *vals);

/* ---- independent oracles (oracle.hpp:73-98) ---- */
int or_bfs_multi_source(uint32_t w, uint32_t h, const uint8_t *occ, const uint8_t *srcmask,
                        uint32_t *hops);
int or_bfs_from(uint32_t w, uint32_t h, const uint8_t *occ, uint32_t row, uint32_t col,
                uint32_t *hops);
int or_dijkstra_octile(uint32_t w, uint32_t h, const uint8_t *occ, const uint8_t *srcmask,
                       int rule, int64_t *axis, int64_t *diag);
uint64_t or_check_activity(uint32_t w, uint32_t h, const uint8_t *occ, const uint32_t *vals,
                           const uint32_t *hops, uint32_t layers, uint32_t *samples_rc,
                           uint32_t max_samples);

/* ---- path extraction (reconstruct.hpp:11-58) ---- */
int or_reconstruct_simple(uint32_t w, uint32_t h, const uint8_t *occ, const uint8_t *srcmask,
                          const uint32_t *vals, uint32_t trow, uint32_t tcol, uint64_t seed,
                          uint32_t *pts_rc, uint64_t cap, uint64_t *npts);
int or_reconstruct_euclidean(uint32_t w, uint32_t h, const uint8_t *occ, const uint8_t *srcmask,
                             const uint32_t *vals, uint32_t trow, uint32_t tcol, int rule,
                             uint32_t *pts_rc, uint64_t cap, uint64_t *npts);
/* occ may be NULL (geometric straighten, reconstruct.hpp:52). In-place safe. */
int or_straighten(const uint32_t *pts_rc, uint64_t n, const uint8_t *occ, uint32_t w,
                  uint32_t h, int rule, uint32_t *out_rc, uint64_t *nout);
void or_path_metrics(const uint32_t *pts_rc, uint64_t n, uint64_t *steps, double *length);

#ifdef __cplusplus
}
#endif
#endif
