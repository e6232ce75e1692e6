/*
 * nbx -- B200 (sm_100a) cluster-pair (nbnxn) neighbour search and
 * short-range non-bonded force: the C ABI.
 *
 * Every entry point replaces one function of the reference Python package
 * clustermd (/root/reference/pkg/src/clustermd); the citation on each
 * declaration names it.  Conventions:
 *   - plain pointers + sizes, no C++ or torch types;
 *   - pointers documented "device" are CUDA device pointers (any allocator,
 *     e.g. torch tensors), "host" are host pointers;
 *   - `stream` is a cudaStream_t passed as void* (0 = legacy default stream);
 *     all work is enqueued on it; functions documented "syncs" wait on it;
 *   - return 0 on success, NBX_ERR_PARAM on a contract violation (the
 *     reference raises ParameterError), NBX_ERR_SINGULAR when an admitted
 *     pair inside the cutoff has r^2 == 0 (SingularityError), NBX_ERR_CUDA
 *     on a CUDA failure; nbx_last_error() describes the last failure.
 *   - grids and lists are opaque, device-resident handles owned by the
 *     library; they are immutable after creation (like the reference's
 *     frozen dataclasses) except for lazily built caches.
 */
#ifndef NBX_H
#define NBX_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum {
  NBX_OK = 0,
  NBX_ERR_PARAM = 1,
  NBX_ERR_SINGULAR = 2,
  NBX_ERR_CUDA = 3
};

enum { NBX_ELEC_CUTOFF = 0, NBX_ELEC_REACTION_FIELD = 1, NBX_ELEC_EWALD = 2 };

enum {
  NBX_FORCE_ENERGY = 1,      /* compute e_lj / e_coulomb (else e_out untouched)         */
  NBX_FORCE_ACCUMULATE = 2,  /* f_out += forces (compute_nonbonded_into semantics)      */
  NBX_FORCE_CLUSTERED = 4,   /* f_out is (n_slots, 3) in slot order, else (n, 3) original */
  NBX_FORCE_CANONICAL = 8,   /* evaluate the canonical CSR rows (generic kernel) even
                                when the grouped fast layout exists (testing aid)      */
  NBX_FORCE_REPRUNE = 16     /* dynamic pruning, rolling prune: after this pass, redo the
                                list's inner masks at this call's positions (GROMACS
                                nstlistPrune); validity is then measured from them  */
};

typedef struct nbx_grid nbx_grid_t;
typedef struct nbx_list nbx_list_t;
typedef struct nbx_dd nbx_dd_t;

typedef struct {
  int32_t n_types;          /* t                                                     */
  const double* lj_table;   /* host, (t, t, 2): [epsilon kJ/mol, sigma nm]            */
  double coulomb_scale;     /* kJ mol^-1 nm e^-2 (model.py:17)                         */
  double r_cut;             /* nm                                                      */
  int32_t shift_potential;  /* subtract the pair energy at r_cut (kernels.py:105-110)  */
  int32_t elec;             /* NBX_ELEC_*                                              */
  double k_rf, c_rf;        /* reaction field (elec == NBX_ELEC_REACTION_FIELD)        */
  double ewald_beta;        /* nm^-1 (elec == NBX_ELEC_EWALD)                          */
} nbx_params_t;

int nbx_version(void);
const char* nbx_last_error(void);
/* instrumentation: kernels launched by this library since load; event
 * timing of the force kernel (enable, then query: total ms + launch count
 * since the last query; the query syncs on the recorded events) */
int64_t nbx_launch_count(void);
void nbx_timing_enable(int32_t on);
int nbx_timing_query(double* total_ms, int64_t* n_launches);

/* ---------------------------------------------------------------- grid
 * Replaces gridder.build_cluster_grid (gridder.py:69-146).  positions:
 * device (n, 3) f64 in original order (wrapped internally, model.py:147).
 * cells = round(sqrt(n / target_occupancy)) computed by the caller exactly
 * as gridder.py:91 does.  Output perm / fill_mask / cell_of_cluster /
 * clustered_positions / bboxes are bit-identical to the reference. */
int nbx_grid_build(const double* positions, int64_t n, const double box[3], int32_t m,
                   int64_t cells, void* stream, nbx_grid_t** out);
/* out = {n, m, cells, n_clusters, n_slots}; syncs */
int nbx_grid_info(const nbx_grid_t* grid, int64_t out[5]);
/* host outputs (any may be NULL): perm (n_slots), inverse_perm (n),
 * fill_mask (n_slots), cell_of_cluster (n_clusters), clustered_positions
 * (n_slots*3), bboxes (n_clusters*6: lo xyz, hi xyz); syncs */
int nbx_grid_download(const nbx_grid_t* grid, int64_t* perm, int64_t* inverse_perm,
                      uint8_t* fill_mask, int64_t* cell_of_cluster, double* clustered_positions,
                      double* bboxes, void* stream);
/* device pointer to the wrapped build-time clustered positions (n_slots, 3) */
const double* nbx_grid_clustered_positions(const nbx_grid_t* grid);
/* gridder.scatter_to_original (gridder.py:149-162): device (n_slots, k) f64
 * -> device (n, k) f64, filler slots dropped */
int nbx_scatter_to_original(const nbx_grid_t* grid, const double* clustered, int32_t k,
                            double* out, void* stream);
void nbx_grid_free(nbx_grid_t* grid);

/* ---------------------------------------------------------------- lists
 * Replaces pairlist.build_pair_list (pairlist.py:147-217): every cluster
 * pair (ci, cj >= ci) whose periodic bounding-box gap is <= r_list, CSR
 * ascending in cj, masks per pairlist.py:106-112.  Errors as :164-175. */
int nbx_pairlist_build(const nbx_grid_t* grid, const double box[3], double r_list, void* stream,
                       nbx_list_t** out);
/* nbx_pairlist_build for one domain of a spatial decomposition: `halo`
 * (device uint8 per particle, original order; NULL = none) marks particles
 * owned by another rank; slot pairs with both particles halo are removed
 * from the masks (their owner computes them).  Otherwise identical. */
int nbx_pairlist_build_ex(const nbx_grid_t* grid, const double box[3], double r_list, const uint8_t* halo,
                          void* stream, nbx_list_t** out);
/* prune_pair_list(build_pair_list(...), positions) in one search (the exact
 * prune criterion applied to each bounding-box hit before it is stored):
 * bit-identical to the two-step result, without the unpruned list.
 * positions: device clustered (n_slots, 3) f64, NULL = the grid's build
 * positions. */
int nbx_pairlist_build_pruned(const nbx_grid_t* grid, const double box[3], double r_list,
                              const double* positions, const uint8_t* halo, void* stream, nbx_list_t** out);
/* Replaces pairlist.prune_pair_list (pairlist.py:242-282): keep rows whose
 * exact FP64 min-image distance over admitted slot pairs is <= r_list, plus
 * every diagonal row.  clustered_positions: device (n_slots, 3) f64. */
int nbx_pairlist_prune(const nbx_list_t* list, const nbx_grid_t* grid,
                       const double* clustered_positions, const double box[3], void* stream,
                       nbx_list_t** out);
/* Extension (dynamic pruning, GROMACS-style inner list): the same pruned
 * list, plus force masks restricted to rows whose FP32 minimum distance at
 * these positions is <= r_inner (conservative one-sided test).  The canonical
 * rows are unchanged; nbx_force uses the inner masks while the maximum
 * displacement since the build satisfies 2 d_max <= r_inner - r_c (checked
 * on the device every call, full masks otherwise).  r_inner = 0: off
 * (== nbx_pairlist_prune).  NBX_ERR_PARAM unless 0 < r_inner <= r_list. */
int nbx_pairlist_prune_inner(const nbx_list_t* list, const nbx_grid_t* grid,
                             const double* clustered_positions, const double box[3], double r_inner,
                             void* stream, nbx_list_t** out);
/* Admitted slot pairs the force kernel evaluates (popcount of the force
 * masks: the inner list when one exists and `inner` != 0, else the
 * canonical list); syncs. */
int nbx_list_force_pairs(nbx_list_t* list, int32_t inner, void* stream, int64_t* n_pairs);
/* out = {n_i_clusters, n_rows, m, n_groups, n_entries}; never syncs.
 * n_rows is -1 until the canonical rows are materialised (lists hold the
 * grouped entries; the canonical CSR is derived from them on first use,
 * nbx_list_rows); n_entries is -1 while a pruned list's live entry count is
 * still only on the device (nbx_list_entries). */
int nbx_list_info(const nbx_list_t* list, int64_t out[5]);
/* live (group, j-cluster) entry count; syncs if not yet known */
int nbx_list_entries(nbx_list_t* list, void* stream, int64_t* n_entries);
/* materialise the canonical CSR rows (pairlist.ClusterPairList offsets /
 * j_idx / masks) if needed and return their count; syncs */
int nbx_list_rows(nbx_list_t* list, void* stream, int64_t* n_rows);
/* host outputs (any may be NULL): offsets (n_i_clusters+1), j_idx (n_rows),
 * masks (n_rows, bit a*m+b of uint64); syncs */
int nbx_list_download(const nbx_list_t* list, int64_t* offsets, int64_t* j_idx, uint64_t* masks,
                      void* stream);
/* Replaces pairlist._build_super_layout (pairlist.py:115-144) for groups of
 * `size` consecutive i-clusters; returns the union entry count; syncs. */
int nbx_super_layout(const nbx_list_t* list, int32_t size, void* stream, int64_t* n_entries);
/* host outputs: super_offsets (n_groups+1), super_j (n_entries),
 * super_pair_idx (n_entries*size, -1 = absent); syncs */
int nbx_super_download(const nbx_list_t* list, int64_t* super_offsets, int64_t* super_j,
                       int64_t* super_pair_idx, void* stream);
/* Extension (rigid water / molecular topologies; the reference masks only
 * fillers and the diagonal, pairlist.py:106-112): clear, in place, every mask
 * bit (canonical and inner force masks) whose two particles belong to the
 * same molecule.  Device int32 arrays: atom_mol (n) molecule id per particle
 * (original order), mol_first (n_mol + 1) / mol_atoms (n) the atoms of each
 * molecule (CSR).  n_removed (host, may be NULL; syncs when given): admitted
 * slot pairs removed.  Cost ~ n x (atoms per molecule) x log(entries per
 * group): a per-particle search of the partners' entries. */
int nbx_list_exclude(nbx_list_t* list, const nbx_grid_t* grid, const int32_t* atom_mol, const int32_t* mol_first,
                     const int32_t* mol_atoms, void* stream, int64_t* n_removed);
/* Extension (list step in one call, for device-resident drivers: run_md,
 * the domain decomposition, bench): nbx_grid_build -> nbx_pairlist_build_ex
 * (halo) -> nbx_list_exclude (when atom_mol != NULL) -> nbx_pairlist_prune_inner
 * at the grid's build positions (flags & NBX_STEP_PRUNE) -> the grouped force
 * layout and its j-cluster transpose (what the first nbx_force call would
 * build).  The same lists as the separate calls, with no host work between
 * the phases (their only host syncs are the grid's cluster count and the
 * search's entry count).  Replaces the rebuild sequence of
 * engine.py:294-334 (_rebuild: build_cluster_grid, build_pair_list,
 * prune_pair_list).  On success *grid_out and *list_out are new handles. */
#define NBX_STEP_PRUNE 1
int nbx_list_step(const double* positions, int64_t n, const double box[3], int32_t m, int64_t cells, double r_list,
                  double r_inner, const uint8_t* halo, const int32_t* atom_mol, const int32_t* mol_first,
                  const int32_t* mol_atoms, int32_t flags, void* stream, nbx_grid_t** grid_out,
                  nbx_list_t** list_out);
/* Per-row diagnostics of pairlist.write_pairs_csv (pairlist.py:349-376):
 * gap_sq[r] = periodic bounding-box gap^2 of row r (gridder.py:165-185),
 * min_d2[r] = exact FP64 minimum admitted slot distance^2 at `positions`
 * (device clustered (n_slots, 3) f64; NULL = the grid's build positions),
 * +inf for rows with no admitted slot pair (_pair_min_dist_sq,
 * pairlist.py:220-239).  Both outputs: device (n_rows) f64, bit-identical to
 * the reference's values.  Materialises the canonical rows (syncs once). */
int nbx_list_diagnostics(nbx_list_t* list, const nbx_grid_t* grid, const double* positions,
                         const double box[3], double* gap_sq, double* min_d2, void* stream);
/* pairlist.interaction_stats / _count_within (pairlist.py:303-346):
 * out = {n_admitted, n_within_cutoff} at clustered_positions; syncs */
int nbx_count_within(const nbx_list_t* list, const double* clustered_positions,
                     const double box[3], double r_cut, void* stream, int64_t out[2]);
void nbx_list_free(nbx_list_t* list);

/* ---------------------------------------------------------------- force
 * Replaces kernels.compute_nonbonded_into (kernels.py:328-396) and its
 * numba kernels (_kernel_blocks :124-221, _kernel_super_blocks :224-312).
 * positions/charges/lj_type: device, original order (n,3) f64, (n) f64,
 * (n) i64.  i_sel: device int32 list of i-clusters (NULL = all).
 * f_out: device f64, (n,3) original order or (n_slots,3) with
 * NBX_FORCE_CLUSTERED.  e_out: device f64[2] = {e_lj, e_coulomb}.
 * bad: device int64[2], set to the clustered slots of a singular pair or -1.
 * FP32 pair arithmetic, FP64 accumulation of energies and of the final
 * forces; results are bit-identical across reruns.  Does not sync; the
 * caller reads bad[] to raise SingularityError. */
int nbx_force(const nbx_list_t* list, const nbx_grid_t* grid, const double* positions,
              const double* charges, const int64_t* lj_type, const nbx_params_t* params,
              const double box[3], const int32_t* i_sel, int64_t n_sel, int32_t flags,
              double* f_out, double* e_out, int64_t* bad, void* stream);

/* ---------------------------------------------------------------- MD step
 * oracle.update_drift (oracle.py:106-123): *out_d2 (device f64) = max over
 * particles of the squared minimum-image displacement cur - ref (FP64,
 * reference operation order; bit-identical). */
int nbx_max_displacement(const double* ref, const double* cur, int64_t n, const double box[3],
                         double* out_d2, void* stream);
/* the same maximum in one launch (the drift guard of every MD / bench step):
 * scratch = 16 B of device memory, zero before the first call and left zero
 * by every call (one caller stream at a time); flags & 1: out = sqrt(max). */
int nbx_max_displacement_ex(const double* ref, const double* cur, int64_t n, const double box[3],
                            uint64_t* scratch, double* out, int32_t flags, void* stream);
/* engine.velocity_verlet_step half steps (engine.py:556-579): v += f*(0.5 dt/m);
 * with move != 0 also x = wrap(x + v dt) (model.py:147-156).  Device arrays,
 * original order. */
int nbx_vv_update(double* x, double* v, const double* f, const double* mass, int64_t n, double dt,
                  int32_t move, const double box[3], void* stream);
/* Extension (rigid 3-site water; the reference has no
 * constraints): molecules are atoms (3k, 3k+1, 3k+2) = (O, H, H) with bond
 * lengths d_oh, d_oh, d_hh.  mode 0 (after the drift of a velocity-Verlet
 * step): SETTLE x (device (3 n_mol, 3) f64, drifted, wrapped) given the
 * constrained positions x_old of the previous step, and v += displacement / dt;
 * mode 1 (after the second half kick): RATTLE velocity stage, v projected so
 * that no bond length changes (x_old unused). */
int nbx_settle(const double* x_old, double* x, double* v, int64_t n_mol, double m_o, double m_h, double d_oh,
               double d_hh, double dt, int32_t mode, const double box[3], void* stream);
/* One velocity-Verlet half for rigid water (3 atoms per molecule, all atoms
 * in molecules), fused with its constraint: phase 0 = half kick + drift +
 * wrap (nbx_vv_update, move) + SETTLE against the pre-drift positions; phase
 * 1 = half kick + RATTLE's velocity stage.  Bit-identical to the separate
 * calls, one launch instead of two or three. */
int nbx_vv_constrained(double* x, double* v, const double* f, const double* mass, int64_t n_mol, double m_o,
                       double m_h, double d_oh, double d_hh, double dt, int32_t phase, const double box[3],
                       void* stream);

/* ---------------------------------------------------------------- domain decomposition
 * Halo exchange of the 1-D slab decomposition (paper_1506_00716_b200/dd.py,
 * the reference's SlabPartition idea engine.py:141-263 turned into ranks):
 * NCCL point-to-point between slab neighbours, enqueued on `stream`.
 * nbx_dd_unique_id on rank 0, broadcast the 128 bytes, nbx_dd_create on
 * every rank (collective).  Local arrays are [home; halo] rows (x 3 f64). */
int nbx_dd_unique_id(uint8_t out[128]);
int nbx_dd_create(const uint8_t uid[128], int32_t nranks, int32_t rank, nbx_dd_t** out);
/* send_local: device int64 indices (local rows) of the home particles sent to rank-1 */
int nbx_dd_set_layout(nbx_dd_t* dd, const int64_t* send_local, int64_t n_send, int64_t n_home,
                      int64_t n_halo, void* stream);
/* coordinates: send_local rows -> rank-1; rows [n_home, n_home+n_halo) <- rank+1 */
int nbx_dd_exchange_positions(nbx_dd_t* dd, double* local_pos, void* stream);
/* forces: rows [n_home, ...) -> rank+1 (owner); forces from rank-1 added to send_local rows */
int nbx_dd_reduce_forces(nbx_dd_t* dd, double* local_f, void* stream);
/* One domain's force pass with its halo exchange (replaces the sequence
 * nbx_dd_exchange_positions -> nbx_force -> nbx_dd_reduce_forces): on the
 * NVLink peer path the exchange overlaps the force kernel -- the work items
 * of the domain list that read no halo coordinate (interior groups, first in
 * the list's work order) run while the halo rows travel; then the halo rows
 * are taken, the boundary items run, and the halo forces are returned.
 * Same arguments and results as nbx_force (no i_sel, no NBX_FORCE_CANONICAL);
 * f_out: device (n_local, 3) in local order.  NCCL path: sequential. */
int nbx_dd_force(nbx_dd_t* dd, const nbx_list_t* list, const nbx_grid_t* grid, double* local_pos,
                 const double* charges, const int64_t* lj_type, const nbx_params_t* params, const double box[3],
                 int32_t flags, double* f_out, double* e_out, int64_t* bad, void* stream);
/* The sequential peer-path force step (halo rows in, then the whole pass)
 * with the halo forces sent as soon as the clusters holding halo particles
 * are reduced (the rest of k_reduce overlaps their transfer); NCCL path:
 * the three calls in sequence.  Same arguments and results as nbx_dd_force. */
int nbx_dd_force_seq(nbx_dd_t* dd, const nbx_list_t* list, const nbx_grid_t* grid, double* local_pos,
                     const double* charges, const int64_t* lj_type, const nbx_params_t* params, const double box[3],
                     int32_t flags, double* f_out, double* e_out, int64_t* bad, void* stream);
int nbx_dd_allreduce_sum(nbx_dd_t* dd, double* buf, int64_t n, void* stream);
/* rebuild-time bookkeeping (dd.SlabDecomposition.assign): from global
 * positions (device n x 3) and host boundaries (N+1), the rank's home / halo
 * ids and send_local (device int64, capacity n, ascending), and on the host
 * counts_out = {n_home, n_halo, n_send, home count of every rank}; also sets
 * the exchange layout.  Syncs. */
int nbx_dd_assign(nbx_dd_t* dd, const double* positions, int64_t n, double box_x, const double* boundaries,
                  double r_comm, int64_t* home, int64_t* halo, int64_t* send_local, int64_t* counts_out,
                  void* stream);
/* nbx_dd_assign plus the rank's local inputs in [home; halo] order: local
 * positions (n_local x 3), charges, types and halo flags (1 for halo rows)
 * gathered from the global arrays into caller device buffers of capacity n
 * (dd.DomainForces.rebuild: one call instead of assign + four gathers). */
int nbx_dd_assign_local(nbx_dd_t* dd, const double* positions, const double* charges, const int64_t* lj_type,
                        int64_t n, double box_x, const double* boundaries, double r_comm, int64_t* home,
                        int64_t* halo, int64_t* send_local, double* local_positions, double* local_charges,
                        int64_t* local_lj_type, uint8_t* local_halo, int64_t* counts_out, void* stream);
/* particle migration at a list step (dd.SlabDecomposition.migrate): for the
 * rank's own particles (device n x 3) the new owner rank (same rule and
 * arithmetic as nbx_dd_assign: np.mod wrap, searchsorted(bnd[1:-1], x,
 * side="right")) and whether the particle lies within r_comm above its new
 * owner's lower boundary (a face particle: halo of the rank below).  Device
 * outputs owner (int32, n) and face (uint8, n); no sync.  Stateless: no
 * nbx_dd_t needed. */
int nbx_dd_classify(const double* positions, int64_t n, double box_x, const double* boundaries, int32_t nranks,
                    double r_comm, int32_t* owner, uint8_t* face, void* stream);
/* global positions from every rank's home rows: one ncclAllGather of
 * (id, x, y, z) records padded to cap >= max home count. */
int nbx_dd_allgather_home(nbx_dd_t* dd, const int64_t* home_ids, const double* home_pos, int64_t n_home,
                          int64_t cap, double* positions_global, void* stream);
/* NVLink peer path for the two per-step exchanges (replaces NCCL send/recv):
 * every rank calls nbx_dd_p2p_alloc (capacity = max halo / face particles,
 * e.g. the global particle count), all-gathers the 64-byte CUDA IPC handles,
 * then nbx_dd_p2p_open with the handles of rank-1 and rank+1.  Afterwards
 * nbx_dd_exchange_positions / nbx_dd_reduce_forces store straight into the
 * neighbour's memory and synchronise through release/acquire flags.
 * Passing NULL handles to nbx_dd_p2p_open switches back to NCCL.
 * nbx_dd_p2p_error reports a timed-out peer wait (syncs). */
int nbx_dd_p2p_alloc(nbx_dd_t* dd, int64_t capacity, uint8_t handle_out[64]);
int nbx_dd_p2p_open(nbx_dd_t* dd, const uint8_t down_handle[64], const uint8_t up_handle[64]);
int nbx_dd_p2p_error(nbx_dd_t* dd, int32_t* out);
/* the same flag as of the last nbx_dd_assign (read by its sync; no sync) */
int nbx_dd_p2p_error_seen(const nbx_dd_t* dd, int32_t* out);
void nbx_dd_free(nbx_dd_t* dd);

/* Exact FP64 scan of every admitted pair for a coincident in-range pair
 * (kernels.py:184-187, 390-395); run when nbx_force reported bad = {-2,-2}
 * (non-finite forces).  out = clustered slots or {-1,-1}; syncs. */
int nbx_find_singular(const nbx_list_t* list, const nbx_grid_t* grid, const double* positions,
                      double r_cut, const double box[3], void* stream, int64_t out[2]);

#ifdef __cplusplus
}
#endif
#endif /* NBX_H */
