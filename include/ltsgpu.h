/* ltsgpu -- B200 (sm_100a) narrow phase for the optimistic local-time-stepping
 * DEM method (arXiv 2309.15417), C ABI.
 *
 * The reference (ltsdem) is pure Python/numpy and has no FFI; its "operator
 * API" for this path is the module `ltsdem.ccd` plus the row kernels in
 * `ltsdem.kernels`.  Each entry point below replaces one of those functions
 * (file:line under /root/reference/pkg/src/ltsdem).  The Python host
 * (`paper_2309_15417_b200/ccd.py`, `kernels.py`) binds them with ctypes and
 * keeps the reference's call surface; INTEGRATION.md shows the binding.
 *
 * Conventions
 *  - Every pointer argument is DEVICE memory owned by the caller unless the
 *    name ends in `_host`.  The library never frees caller memory.
 *  - Every call is ordered on `stream` (a cudaStream_t, NULL = legacy default)
 *    and re-entrant; all scratch lives in an explicit workspace handle.
 *  - Arrays of 3-vectors are row-major (n, 3) float64; triangles are
 *    (n, 3, 3) float64 (corner-major), exactly numpy's C layout.
 *  - Return value: LTSG_OK or an error code; ltsg_last_error() gives a
 *    thread-local message.  On LTSG_ECAPACITY the caller grows its output
 *    buffers (sizes reported in the out struct) and calls again.
 *  - All arithmetic is IEEE float64 with the reference's rounding order, so
 *    static (dt = 0) results are bit-identical to the reference.
 */
#ifndef LTSGPU_H
#define LTSGPU_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define LTSG_OK 0
#define LTSG_EINVAL 1
#define LTSG_ECUDA 2
#define LTSG_ECAPACITY 3
#define LTSG_ENOMEM 4 /* cudaMalloc failed inside the budget: a real out-of-memory, not retried */

const char* ltsg_last_error(void);
int ltsg_version(void);

/* kernels.point_triangle_closest (kernels.py:23-75): per row, the closest
 * point on triangle (a, b, c) to p and its distance.  `closest` may be NULL. */
int ltsg_point_triangle_closest(const double* p, const double* a, const double* b,
                                const double* c, int64_t n, double* dist, double* closest,
                                void* stream);

/* kernels.segment_segment_closest (kernels.py:78-115).  c1/c2 may be NULL. */
int ltsg_segment_segment_closest(const double* p1, const double* q1, const double* p2,
                                 const double* q2, int64_t n, double* dist, double* c1,
                                 double* c2, void* stream);

/* ccd._feature_distances (ccd.py:135-153): row-wise 15-feature distance of
 * triangle pairs tri_a[i], tri_b[i], each (n, 3, 3). */
int ltsg_feature_distances(const double* tri_a, const double* tri_b, int64_t n, double* dist,
                           void* stream);

/* ccd._closest_feature (ccd.py:156-174) per row: distance and witness points
 * pa (on tri_a) and pb (on tri_b), (n, 3) each. */
int ltsg_closest_feature(const double* tri_a, const double* tri_b, int64_t n, double* dist,
                         double* pa, double* pb, void* stream);

/* kernels.triangle_overlap_centroid (kernels.py:138-201) per row; has[i] = 0
 * where the reference returns None. */
int ltsg_overlap_centroid(const double* tri_a, const double* tri_b, const double* normal,
                          int64_t n, double* centroid, int32_t* has, void* stream);

/* ---------------------------------------------------------------- search
 *
 * One call runs ccd._search (ccd.py:373-487) for a batch of independent
 * problems: a problem is one `pair_earliest_contact` call (one body pair,
 * ccd.py:490-502) or one `compute_effective_dt` cluster (several pairs
 * sharing one bound, ccd.py:505-524).  It also builds the contact records
 * (_make_contact, ccd.py:183-213) and fuses them (filter_contacts,
 * ccd.py:527-577).
 *
 * Packed scene (device, built by the host packer):
 *  tris       n_tris x 16 float64 triangle records: 9 body-frame corners,
 *             epsilon, arm (max corner norm), (int32 first child, int32 child
 *             count) packed into slot 11, and the body-frame bounding sphere
 *             (centroid in 12..14, radius in 15, -1 for slivers).  Each tree level
 *             is stored so that a parent's children form a contiguous range
 *             of the next finer level.
 *  tri_orig   n_tris int32: the triangle's index in the reference tree level
 *             (reported as tri_a / tri_b).
 *  body_state n_bodies x 16 float64: position[3], velocity[3], rotation
 *             quaternion [w,x,y,z], angular_velocity[3], static flag, 2 pad.
 *  body_levels n_bodies x 18 int64: n_levels, id, then 8 level record
 *             offsets and 8 level sizes.
 *  pair_body  n_pairs x 2 int32 body slots; pair_problem n_pairs int32;
 *  pair_group n_pairs int32: rank of (body_a id, body_b id) among the distinct
 *             id pairs of the pair's problem (fusion groups, ccd.py:535-539).
 *  problem_dt / problem_tbase  n_problems float64.
 */
typedef struct {
  const double* tris;
  const int32_t* tri_orig;
  int64_t n_tris;
  const double* body_state;
  const int64_t* body_levels;
  int32_t n_bodies;
  int32_t n_problems;
  const int32_t* pair_body;
  const int32_t* pair_problem;
  const int32_t* pair_group;
  int64_t n_pairs;
  const double* problem_dt;
  const double* problem_tbase;
  double widen;
  int32_t exhaustive;
  int32_t max_children;  /* max children per surrogate triangle (fanout) */
} ltsg_scene;

/* ---------------------------------------------------------------- compact tree upload
 *
 * The triangle records of `ltsg_scene.tris` rebuilt on the device from a
 * compact host image (about 1/3 of the record bytes): the fine level as
 * deduplicated vertices plus three vertex indices per triangle (the
 * reference's level-0 corners are rows of the mesh vertex array,
 * body.py:70-72 / surrogate.py:91, so the dedup is exact), the coarse
 * levels as 9 corners, epsilon per record (or one value for a constant
 * fine level, surrogate.py:89), and (first child, count) per coarse
 * record.  The derived slots are computed on the device: arm with the
 * reference's norm order (ccd._Motion.arm, ccd.py:108-114) and the cull
 * sphere.  Replaces the host-side record build of the packer; the result is
 * bit-identical to it in slots 0-11.
 *
 * Per tree (table row of 8 int64):
 *   rec_off   first record of the tree in `tris_out`
 *   n_fine    level-0 record count (records rec_off .. rec_off+n_fine-1)
 *   n_coarse  coarse record count (the records after the fine ones)
 *   vert_off  first vertex of the tree in `verts`
 *   vidx_off  first fine record of the tree in `vidx` (3 int32 each; tree-local vertex ids)
 *   coarse_off first coarse record of the tree in `coarse` (9 doubles each) and `kids` (2 int32 each)
 *   eps_off   first epsilon of the tree in `eps`
 *   eps_mode  1: one epsilon per record; 0: eps[eps_off] for every fine record,
 *             then one per coarse record */
typedef struct {
  const double* verts;
  const int32_t* vidx;
  const double* coarse;
  const double* eps;
  const int32_t* kids;
  const int64_t* table;
  int32_t n_trees;
  int32_t pad;
} ltsg_tree_upload;

int ltsg_unpack_trees(const ltsg_tree_upload* up, double* tris_out, void* stream);

/* Per-problem results and the contact lists (device buffers, caller-owned).
 * Contacts are SoA; `fused_*` are the filter_contacts output grouped by
 * problem (problem p's fused contacts are [fused_offset[p], fused_offset[p+1]));
 * `raw_*` (optional, may be NULL) are the pre-fusion records. */
typedef struct {
  double* dt;             /* n_problems */
  double* first_contact;  /* n_problems; valid where collision */
  int32_t* collision;     /* n_problems */
  int64_t* fused_offset;  /* n_problems + 1 */
  int64_t capacity;       /* contact capacity of each list below */
  int32_t* body_a;
  int32_t* body_b;
  double* position;       /* (capacity, 3) */
  double* normal;         /* (capacity, 3) */
  double* depth;
  double* t;
  int32_t* tri_a;
  int32_t* tri_b;
  double* threshold;
  int32_t* problem;       /* problem of each fused contact */
  /* optional raw (pre-fusion) records */
  int32_t* raw_problem;
  int32_t* raw_body_a;
  int32_t* raw_body_b;
  double* raw_position;
  double* raw_normal;
  double* raw_depth;
  double* raw_t;
  int32_t* raw_tri_a;
  int32_t* raw_tri_b;
  double* raw_threshold;
  /* filled by the call (host-visible scalars) */
  int64_t n_fused;
  int64_t n_raw;
  int64_t rows_screen;    /* 15-feature rows of the multiscale screen (= reference) */
  int64_t rows_zoom;      /* zoom rows the reference would evaluate */
  int64_t rows_bisect;    /* bisection rows */
  int64_t rows_executed;  /* rows actually evaluated on the device */
  int64_t candidates;     /* candidates screened over all levels */
  int32_t generations;
  int32_t launches;       /* kernels launched by the call */
  double ms_screen;       /* device time of the screen kernels (CUDA events) */
  double ms_refine;       /* zoom + bisection */
  double ms_contacts;     /* records, contacts, fusion */
  int64_t rows_screen_exact; /* screen rows that ran the exact 15-feature distance
                                (the rest were settled by the certified culls) */
  double ms_exact;        /* device time of the exact-distance kernels (k_screen_static / k_mexact) */
  double ms_expand;       /* device time of the child expansion + culls (static) / decisions (moving) */
  int64_t rows_bound;     /* rows that survived the culls and were decided by the certified FP32
                             upper bound instead of the exact distance (rows_screen_exact excludes them) */
} ltsg_result;

typedef struct ltsg_workspace ltsg_workspace;

/* Scratch owner for ltsg_search: grows on demand, reused across calls.  One
 * workspace per concurrent stream.  All workspaces of the process draw from
 * one pool of 75% of the device memory free at the first allocation, so
 * concurrent engine threads cannot jointly exceed the device; `budget_bytes`
 * additionally caps this workspace (0 = pool only).  Beyond either limit a
 * call returns LTSG_ECAPACITY (the host splits the batch); a cudaMalloc
 * failure inside them returns LTSG_ENOMEM. */
ltsg_workspace* ltsg_workspace_create(int64_t budget_bytes);
void ltsg_workspace_destroy(ltsg_workspace* ws);
int64_t ltsg_workspace_bytes(const ltsg_workspace* ws);

/* Run the batched search.  Blocks the calling thread until `stream` has
 * finished the call (the traversal reads frontier sizes back each level). */
int ltsg_search(const ltsg_scene* scene, ltsg_result* out, ltsg_workspace* ws, void* stream);

/* ccd.filter_contacts (ccd.py:527-577) on caller-provided raw contacts: the
 * raw_* arrays of `io` (n_raw entries) are the input, group_key[i] =
 * (problem << 32) | rank of (body_a, body_b) within the problem; the fused
 * outputs and fused_offset of `io` are written.  On entry io->n_raw must hold
 * the number of problems. */
int ltsg_fuse_contacts(ltsg_result* io, int64_t n_raw, const uint64_t* group_key,
                       ltsg_workspace* ws, void* stream);

/* Roofline measurement of the 15-feature distance: every fine x fine row of
 * every pair at tau = 0 evaluated exactly (no cull, no traversal).  Returns
 * the row count, the rows within h + 1e-9 and the kernel's device time. */
int ltsg_exhaustive_rows(const ltsg_scene* scene, int64_t* rows, int64_t* hits, double* ms,
                         ltsg_workspace* ws, void* stream);

/* The same rows with every distance written out: out_dist (device, float64)
 * receives, pair after pair, the na x nb fine rows of each pair row-major in
 * world-record order (record i of body a, record j of body b; tri_orig maps
 * records to reference triangle indices).  Each value is
 * ccd._feature_distances (ccd.py:135-153) of that row at tau = 0.  *rows
 * receives the total row count.  Parity/validation entry point. */
int ltsg_exhaustive_distances(const ltsg_scene* scene, double* out_dist, int64_t* rows,
                              ltsg_workspace* ws, void* stream);

/* FP64 pipe microbenchmark: independent DFMA chains on every SM; reports
 * the achieved FP64 FLOP/s (2 per DFMA) -- the roofline denominator. */
int ltsg_fp64_peak(double* tflops, double* ms, void* stream);


/* ---------------------------------------------------------------------------
 * Space-time broad phase: ltsdem.broadphase.build_collision_graph
 * (broadphase.py:198-252), the step before the narrow phase.  It produces the
 * candidate pairs (edges) and static links the narrow phase screens.
 *
 * particle: (n_particles, 28) float64 records, particles in ascending id
 *   order: [0:3] old.position [3:7] old.rotation [7] old.t
 *          [8:11] current.position [11:15] current.rotation [15] current.t
 *          [16:19] current.velocity [19:22] current.angular_velocity
 *          [22:25] sphere.center (body frame) [25] sphere.radius [26:28] unused
 *   (the fields _Trajectory.of_particle reads, :83-95, with particle_dt's
 *   timeline stamps, :46-50).
 * statics: (n_statics, 4) float64 world spheres (center, radius) in ascending
 *   static-id order (_Trajectory.of_static, :97-99).
 * Body index i < n_particles is particle i, n_particles + k is static k; the
 * reference's `ids = pids + sids` (:220).
 */
typedef struct {
  const double* particle;
  const double* statics;
  int32_t n_particles;
  int32_t n_statics;
  double dt_max;  /* TimeStepPolicy.dt_max (:36) */
  double growth;  /* TimeStepPolicy.growth (:37) */
} ltsg_broad_input;

typedef struct {
  double* dts;        /* n_particles: particle_dt per particle (graph.dts); may be NULL */
  int32_t* edge;      /* (cap_edges, 2) particle indices a < b, in the reference's edge-dict order */
  double* window;     /* (cap_edges, 2) the pair window of each edge (graph.edges values) */
  int32_t* link;      /* (cap_links, 2) (particle index, static index), sorted: graph.static_links */
  int64_t cap_edges;
  int64_t cap_links;
  /* filled by the call */
  int64_t n_edges;
  int64_t n_links;
  int64_t candidates; /* body pairs that passed Check 1 (the boxes overlap) */
  int32_t launches;
  int32_t pad;
  double ms;          /* device time of the call (CUDA events) */
} ltsg_broad_output;

/* Build the collision graph.  Blocks until `stream` has finished the call
 * (the output counts are read back).  LTSG_ECAPACITY when n_edges/n_links
 * exceed the capacities: the counts are set, grow and call again. */
int ltsg_broadphase(const ltsg_broad_input* in, ltsg_broad_output* out, ltsg_workspace* ws, void* stream);

/* check_spacetime_tube / _min_distance_over_window (broadphase.py:128-158) on
 * explicit trajectory rows: t (n,3) knot times, c (n,3,3) centres, r (n,)
 * radius, nt (n,) knot count (3 for a particle, 1 for a static); win (n,2).
 * Writes the minimum centre distance and the Check-2 verdict per row. */
int ltsg_tube_rows(const double* t1, const double* c1, const double* r1, const int32_t* nt1,
                   const double* t2, const double* c2, const double* r2, const int32_t* nt2,
                   const double* win, int64_t n, double* dist, int32_t* hit, void* stream);

/* ---------------------------------------------------------------------------
 * Contact consumers: ltsdem.contacts (contacts.py), the step after the narrow
 * phase, for many clusters ("problems") in one launch.  A dynamic body may
 * appear in the contacts of one problem only (engine clusters are disjoint).
 *
 * body: (n_bodies, 24) float64 records of the bodies' current snapshots:
 *   [0:3] position [3:6] velocity [6:10] rotation [10:13] angular_velocity
 *   [13] t [14] 1 / mass [15:24] body-frame inverse inertia (row-major)
 *   (what _contact_arm reads, contacts.py:100-111, body.py:39-41).
 * Contacts of problem p are [contact_offset[p], contact_offset[p+1]) in the
 * caller's order; side (n, 2) holds each side's body index, -1 for a static.
 */
typedef struct {
  const double* body;
  int32_t n_bodies;
  int32_t n_problems;
  const int64_t* contact_offset; /* n_problems + 1 */
  const int32_t* side;           /* (n_contacts, 2) */
  const double* position;        /* (n_contacts, 3) ContactPoint.position */
  const double* normal;          /* (n_contacts, 3) ContactPoint.normal */
  const double* t;               /* (n_contacts) ContactPoint.t */
  int64_t n_contacts;
  double restitution, friction, relaxation, penalty, threshold; /* SolverConfig (contacts.py:26-33) */
  int32_t max_iterations;
  int32_t pad;
} ltsg_solve_input;

typedef struct {
  double* velocity;          /* (n_bodies, 3) post-impulse velocity of every touched body */
  double* angular_velocity;  /* (n_bodies, 3) */
  int32_t* touched;          /* (n_bodies) 1 if the body is a dynamic side of some contact */
  double* normal_impulse;    /* (n_contacts) ImpulseSolution.normal_impulses */
  double* friction_impulse;  /* (n_contacts, 3) ImpulseSolution.friction_impulses */
  int32_t* color;            /* (n_contacts) colour class (color_contact_graph) */
  int32_t* iterations;       /* (n_problems) */
  int32_t* converged;        /* (n_problems) */
  int32_t launches;
  int32_t pad;
  double ms;                 /* device time of the call */
} ltsg_solve_output;

/* solve_impulses (contacts.py:114-198) per problem, with color_contact_graph
 * (:58-78).  Blocks until `stream` has finished the call. */
int ltsg_solve_impulses(const ltsg_solve_input* in, ltsg_solve_output* out, ltsg_workspace* ws, void* stream);

typedef struct {
  const double* body;            /* (n_bodies, 24) as ltsg_solve_input */
  int32_t n_bodies;
  int32_t n_problems;
  const int64_t* member_offset;  /* n_problems + 1 */
  const int32_t* member;         /* body indices of each problem's cluster members */
  const double* t_new;           /* (n_problems) cluster.t_current + result.dt */
  const int64_t* contact_offset; /* n_problems + 1: the committed contacts */
  const int32_t* side;           /* (n_contacts, 2) body index or -1 */
  const int64_t* id;             /* (n_contacts, 2) body ids (ContactPoint.body_a/b; statics negative) */
  const double* normal;          /* (n_contacts, 3) */
  const double* t;               /* (n_contacts) */
  const double* depth;           /* (n_contacts) */
  int64_t n_contacts;
  const double* velocity;        /* solution (ltsg_solve_output), or NULL for none */
  const double* angular_velocity;
  const int32_t* touched;
  double beta;                   /* SolverConfig.beta */
  const double* new_state_in;    /* NULL: integrate; else (n_bodies, 14) new snapshots to start from
                                    (apply_separation alone, contacts.py:256-285) */
  int32_t separate;              /* 1: apply_separation after the integration */
  int32_t pad;
} ltsg_integrate_input;

/* integrate_cluster (contacts.py:225-253) then apply_separation (:256-285)
 * per problem: new_state (n_bodies, 14) receives each member's prospective
 * snapshot [0:3] position [3:6] velocity [6:10] rotation [10:13]
 * angular_velocity [13] t (rows of non-members are untouched). */
int ltsg_integrate(const ltsg_integrate_input* in, double* new_state, ltsg_workspace* ws, void* stream);

/* ---------------------------------------------------------------------------
 * Surrogate-tree construction: ltsdem.surrogate.build_surrogate_tree
 * (surrogate.py:71-119, with _fit_parent_triangle :49-68 and
 * kernels.morton_order kernels.py:118-135) for many meshes in one call --
 * the narrow phase's input format (ltsg_scene.tris / ltsg_unpack_trees).
 *
 * All records of all meshes live in one table: `rec` (n_records, 9) float64
 * corners, `eps` (n_records) halo widths, `kids` (n_records) int32.  The
 * caller lays the levels out (level l+1 of a mesh has ceil(size_l / fanout)
 * records; coarsening stops at one record or max_levels), fills the level-0
 * rows of `rec` and `eps`, and describes each (mesh, coarse level) as a row
 * of the device table `steps` (n_steps, 6) int64:
 *   [in_off, n_in, out_off, n_out, key_off, group_off]
 * in_off/n_in: the finer level's records; out_off/n_out: the coarse level's;
 * key_off/group_off: prefix sums of n_in / n_out over the rows of the same
 * coarse level.  Rows are grouped by coarse level; rows of level l (1-based)
 * are [level_steps[l-1], level_steps[l]) and level_keys / level_groups (host
 * arrays, n_levels each) hold the sums of n_in / n_out over them.
 * The call writes every coarse record's corners and epsilon and, for every
 * record with a parent, kids[in_off + fanout*g + j] = the j-th entry of
 * parent g's sorted child list (surrogate.py:115).  Bit-identical to the
 * reference with numpy's bundled OpenBLAS/LAPACK (SkylakeX kernels); see
 * csrc/lapack3.cuh.  fanout 2..8.  Blocks until `stream` has finished. */
typedef struct {
  double* rec;
  double* eps;
  int32_t* kids;
  const int64_t* steps;        /* device */
  const int64_t* level_steps;  /* host, n_levels + 1 */
  const int64_t* level_keys;   /* host, n_levels */
  const int64_t* level_groups; /* host, n_levels */
  int32_t n_levels;
  int32_t fanout;
  int32_t launches;            /* filled by the call */
  int32_t pad;
} ltsg_tree_build;

int ltsg_build_trees(ltsg_tree_build* b, ltsg_workspace* ws, void* stream);

#ifdef __cplusplus
}
#endif

#endif
