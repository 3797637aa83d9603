/* dlb — B200-native collide-and-stream for the dolb lattice Boltzmann solver.
 *
 * C ABI of libdlb_b200.so. Plain pointers and sizes only. Conventions follow
 * the reference C interface (proj/include/dolb/dolb.h:1-32, proj/src/capi.cpp:13-39):
 * every call returns DLB_OK (0) or a nonzero status; dlb_last_error() (thread
 * local) describes the failure; handles are opaque and released by their free
 * function. Status values are numerically identical to dolb_status.
 *
 * What each group replaces in the reference (file:line under /root/reference/proj):
 *   dlb_chain_* / dlb_registry_*  DynamicsRegistry + chain strings
 *                                 (include/dolb/accelerated_lattice.hpp:32-79,
 *                                  src/accelerated_lattice.cpp:10-84, src/chain.cpp:38-230)
 *   dlb_lattice_*                 AcceleratedBlock<T> + collide_and_stream<T> +
 *                                 MultiBlockRun<T>::{fill,advance,gather_populations}
 *                                 (include/dolb/accelerated_lattice.hpp:86-127,
 *                                  include/dolb/multiblock.hpp:119-159)
 *   dlb_lattice_link_* / _ipc     Transport + envelope exchange of one z-slab
 *                                 (include/dolb/multiblock.hpp:93-109, src/multiblock.cpp:289-355)
 *   dlb_collide_and_stream        collide_and_stream<T>(AcceleratedBlock<T>&, registry,
 *                                 recipes, dispatch, nthreads) on HOST buffers
 *                                 (include/dolb/accelerated_lattice.hpp:124-127)
 *   dlb_lattice_reduce* /         diag::tree_sum / kinetic_energy / vorticity_fd8 / enstrophy
 *   dlb_tree_* / _snapshot_*      and Driver::sample / porous_extras on the resident state
 *                                 (src/diagnostics.cpp:10-131, src/runner.cpp:346-448)
 *   dlb_case_*                    init_tgv / init_cavity / init_porous input generators
 *                                 (include/dolb/cases.hpp:96-98, src/cases.cpp:127-260)
 */
#ifndef DLB_H
#define DLB_H

#include <stddef.h>
#include <stdint.h>

#define DLB_API __attribute__((visibility("default")))

#ifdef __cplusplus
extern "C" {
#endif

typedef enum dlb_status {
    DLB_OK = 0,
    DLB_ERROR_INVALID_ARGUMENT = 1,
    DLB_ERROR_CONFIG = 2,
    DLB_ERROR_IO = 3,
    DLB_ERROR_DISPATCH = 4,
    DLB_ERROR_EXCHANGE = 5,
    DLB_ERROR_INTERNAL = 6, /* includes CUDA failures; no CPU fallback exists */
} dlb_status;

enum { DLB_LAYOUT_TWO_POP = 0, DLB_LAYOUT_AA = 1 };
enum { DLB_ARITH_EXACT = 0, /* reference operation order, no FMA: bit-identical   */
       DLB_ARITH_FAST = 1 };  /* FMA contraction allowed (fp64 drift <= 1e-12 rel) */

DLB_API const char* dlb_version(void);
DLB_API const char* dlb_last_error(void);

/* ---- dynamics chains (src/chain.cpp:38-151) -------------------------------- */
/* Parse + validate a chain string and write its canonical rendering. */
DLB_API dlb_status dlb_chain_canonical(const char* chain, char* buf, size_t cap, size_t* len_out);

/* ---- registry (src/accelerated_lattice.cpp:10-84) -------------------------- */
typedef struct dlb_registry dlb_registry;
DLB_API dlb_status dlb_registry_new(dlb_registry** out);
DLB_API void dlb_registry_free(dlb_registry* reg);
/* register_chain: chain string + its serialize_params record (chain.cpp:153-186).
 * Idempotent for identical (chain, params); rejects omega outside (0, 2). */
DLB_API dlb_status dlb_registry_register(dlb_registry* reg, const char* chain,
                                         const double* params, size_t n_params,
                                         int32_t* slot_out);
DLB_API dlb_status dlb_registry_tag_for(const dlb_registry* reg, const char* chain,
                                        int32_t* tag_out);
DLB_API dlb_status dlb_registry_chain_for(const dlb_registry* reg, int32_t tag, char* buf,
                                          size_t cap, size_t* len_out);
DLB_API dlb_status dlb_registry_tag_of_slot(const dlb_registry* reg, int32_t slot,
                                            int32_t* tag_out);
DLB_API dlb_status dlb_registry_counts(const dlb_registry* reg, int32_t* num_tags,
                                       int32_t* num_instances);
DLB_API dlb_status dlb_registry_slot_params(const dlb_registry* reg, int32_t slot, double* buf,
                                            size_t cap, size_t* len_out);

/* ---- device lattice: one z-slab of the domain on one GPU -------------------- */
typedef struct dlb_lattice dlb_lattice;
typedef struct dlb_lattice_desc {
    int64_t dims[3];         /* interior cells of this slab (x, y, z) */
    int32_t periodic[3];     /* global periodicity of the domain */
    int32_t q;               /* 19 or 27 */
    int32_t precision_bits;  /* 32 or 64 */
    int32_t layout;          /* DLB_LAYOUT_* */
    int32_t arith;           /* DLB_ARITH_* */
    int32_t device;          /* CUDA ordinal */
    int64_t z_origin;        /* global z index of the slab's first interior plane */
    int64_t global_nz;       /* global z extent (== dims[2] for a single slab) */
    int32_t flags;           /* DLB_FLAG_* */
    int32_t reserved;
} dlb_lattice_desc;

/* Masked porous variant: NoDynamics cells are neither loaded nor stored, at the
 * granularity of x-aligned groups of one 32-B segment per direction array (a
 * group moves nothing only when all its cells are NoDynamics; the NoDynamics
 * cells of a mixed group run their dense update). Precondition (checked by
 * dlb_lattice_set_slots, DLB_ERROR_CONFIG otherwise): no collision cell has a
 * NoDynamics neighbour -- a solid cell next to fluid must be BounceBack, as the
 * reference's porous setup assigns (cases.cpp:239-249; z neighbours in other
 * slabs are not checked). Then the skipped values are never consumed by a
 * collision cell (bounce-back cells only return a cell's own populations to
 * it), so every collision cell stays bit-identical to the reference
 * (SURVEY.md A.4). Works on single slabs and z-slabs. */
#define DLB_FLAG_SKIP_NODYNAMICS 1
/* Use a TMA-staged dense kernel for single-slab two-population lattices:
 * k_tmablk on uniform lattices (one 2-D tensor box of 256 x R rows per
 * direction and work unit), else the row-staged k_tmarow (each direction's
 * whole source row as 3-D tensor-map boxes), both into 2-stage mbarrier rings
 * (DLB_TMA_ROW=0 selects the box-tiled k_tma). Opt-in: on B200 they reach
 * 0.70-0.86 of the copy roofline against 0.94-0.99 for the default plain-load
 * kernel (profiles/r01_summary.md). */
#define DLB_FLAG_TMA 2
/* Sparse porous variant (single slab): per-slot, row-major cell lists, one
 * launch per dynamics kind; NoDynamics cells are not listed and wall cells
 * move only the links that feed fluid cells. Implies the masked sweep where
 * lists do not apply (z-slabs, AA). Slower than the masked sweep on B200
 * (profiles/r01_summary.md): kept for comparison. */
#define DLB_FLAG_SPARSE_LISTS 4

DLB_API dlb_status dlb_lattice_create(const dlb_lattice_desc* desc, const dlb_registry* reg,
                                      dlb_lattice** out);
DLB_API void dlb_lattice_free(dlb_lattice* lat);
/* Registry instance slot of every interior cell, x fastest (MultiBlockRun::fill's slot_of). */
DLB_API dlb_status dlb_lattice_set_slots(dlb_lattice* lat, const int32_t* slots);
DLB_API dlb_status dlb_lattice_set_uniform_slot(dlb_lattice* lat, int32_t slot);
/* Dispatch set (accelerated_lattice.hpp:63-79). A present tag outside it makes
 * dlb_lattice_step fail with DLB_ERROR_DISPATCH before any cell is written. */
DLB_API dlb_status dlb_lattice_set_dispatch(dlb_lattice* lat, const int32_t* tags, size_t n);
/* Stored state := equilibrium2<T>(T(rho), T(u)) per cell (multiblock.cpp:278-281). */
DLB_API dlb_status dlb_lattice_fill_equilibrium(dlb_lattice* lat, const double* rho,
                                                const double* ux, const double* uy,
                                                const double* uz);
/* Taylor-Green initial state of an L^3 box (cases.cpp:145-156), built on the device. */
DLB_API dlb_status dlb_lattice_fill_tgv(dlb_lattice* lat, int64_t L, double u_inf);
/* Canonical populations: q arrays of nx*ny*nz doubles, direction-major, x fastest
 * (MultiBlockRun::gather_populations order, multiblock.cpp:421-441). */
DLB_API dlb_status dlb_lattice_upload_populations(dlb_lattice* lat, const double* canon);
DLB_API dlb_status dlb_lattice_download_populations(dlb_lattice* lat, double* canon);
/* Same, in the storage precision (float for 32-bit lattices). */
DLB_API dlb_status dlb_lattice_download_raw(dlb_lattice* lat, void* canon);
/* MultiBlockRun::gather_macroscopic (multiblock.cpp:443-484) for this slab:
 * per cell (x fastest) rho and u in double; Collide cells compute_rho_u of the
 * populations converted to double, moving walls rho = 1 and their wall velocity,
 * other cells rho = 1, u = 0. */
DLB_API dlb_status dlb_lattice_gather_macroscopic(dlb_lattice* lat, double* rho, double* ux,
                                                  double* uy, double* uz);
/* Exact, order-independent checksum of the canonical state (q values): for each
 * direction i, sum over cells of bits(double(f_i) + 0.0) * (global cell index + 1)
 * modulo 2^64. Independent of layout and decomposition (slab sums add up), so
 * full-size runs can be compared with the reference without moving the state. */
DLB_API dlb_status dlb_lattice_checksum(dlb_lattice* lat, uint64_t* per_direction);
/* The same over the cells whose chain is not NoDynamics only (the cells the
 * masked porous sweep keeps current). */
DLB_API dlb_status dlb_lattice_checksum_active(dlb_lattice* lat, uint64_t* per_direction);
/* Advance nsteps (asynchronous on the lattice stream; includes the halo exchange). */
DLB_API dlb_status dlb_lattice_step(dlb_lattice* lat, int64_t nsteps);
DLB_API dlb_status dlb_lattice_synchronize(dlb_lattice* lat);
DLB_API dlb_status dlb_lattice_stream(dlb_lattice* lat, void** stream_out);
DLB_API dlb_status dlb_lattice_steps_done(dlb_lattice* lat, int64_t* steps_out);
/* Algorithmic bytes per cell update (2*q*sizeof(T) + slot bytes), device bytes held,
 * and kernel launches per step (for bench accounting). */
DLB_API dlb_status dlb_lattice_traffic(dlb_lattice* lat, int64_t* bytes_per_cell,
                                       int64_t* device_bytes, int32_t* launches_per_step);
/* Algorithmic HBM bytes one step moves (dense: cells * bytes_per_cell; sparse
 * porous mode: fluid cells 2*q*s + 8 B list entry, wall cells only the links that
 * feed fluid cells). */
DLB_API dlb_status dlb_lattice_step_bytes(dlb_lattice* lat, int64_t* bytes_out);
/* Time nsteps with CUDA events recorded on the lattice stream (milliseconds). */
DLB_API dlb_status dlb_lattice_time_steps(dlb_lattice* lat, int64_t nsteps, double* ms_out);
/* Name of the kernel instantiation selected for the present dynamics. */
DLB_API dlb_status dlb_lattice_kernel_name(dlb_lattice* lat, char* buf, size_t cap,
                                           size_t* len_out);

/* ---- z-slab halo exchange over peer memory ---------------------------------- */
/* Same process (any devices with peer access, or one device): the top plane of
 * `lower` feeds the bottom ghost plane of `upper` and vice versa. Both slabs
 * must share the layout. AA slabs (one in-place array per slab) may be linked
 * too: their odd steps store across the faces into the neighbour's boundary
 * plane, so linking clears an AA slab's state (fill / upload after linking,
 * then exchange, as MultiBlockRun does). */
DLB_API dlb_status dlb_lattice_link_local(dlb_lattice* lower, dlb_lattice* upper);
/* Envelope exchange only (MultiBlockRun::exchange, multiblock.hpp:142-143):
 * copy this slab's boundary planes into the linked neighbours' ghost planes of
 * the current state. Call on every slab after filling / uploading the state and
 * before the first step (steps then push the halo themselves). */
DLB_API dlb_status dlb_lattice_exchange(dlb_lattice* lat);
/* The same for several slabs of ONE process: waits for all of them first. */
DLB_API dlb_status dlb_lattices_exchange(dlb_lattice** lats, size_t n);
/* Halo wait limit of a linked slab (default 20 s, or DLB_HALO_TIMEOUT_MS). A
 * neighbour that has not finished the previous step's boundary planes within
 * it fails the step: nothing of that step or of any later queued step is
 * written, the next synchronize / step / download reports DLB_ERROR_EXCHANGE
 * (the reference's lost-message ExchangeError, multiblock.cpp:305-345), and the
 * lattice is left at its last completed step. dlb_lattice_exchange clears the
 * error once the slabs are back at one step count. */
DLB_API dlb_status dlb_lattice_set_halo_timeout(dlb_lattice* lat, double seconds);
/* Link state of a slab: *lower / *upper = 0 not linked, 1 linked to a slab on
 * the same GPU, 2 linked to a slab on another GPU (peer memory over NVLink);
 * *halo_bytes_per_step = population bytes this slab pushes into its
 * neighbours' ghost planes per step (nx * ny * 5 (D3Q19) or 9 (D3Q27) links
 * per linked face). */
DLB_API dlb_status dlb_lattice_links(dlb_lattice* lat, int32_t* lower, int32_t* upper,
                                     int64_t* halo_bytes_per_step);
/* With DLB_TRACE_HALO set (CUDA graphs then off): timeline of the linked steps
 * since the last call, ms from the first event, 5 values per step (halo wait
 * begin / end and boundary-launch end on the halo stream, interior launch
 * begin / end on the main stream). out may be NULL to query the count. */
DLB_API dlb_status dlb_lattice_halo_trace(dlb_lattice* lat, double* out, size_t cap, size_t* n_out);
/* Across processes: export an opaque blob (CUDA IPC handles), ship it with any
 * transport (e.g. torch.distributed), link it as the lower (side 0) or upper
 * (side 1) neighbour. */
DLB_API dlb_status dlb_lattice_export_ipc(dlb_lattice* lat, void* blob, size_t cap,
                                          size_t* len_out);
DLB_API dlb_status dlb_lattice_link_ipc(dlb_lattice* lat, int32_t side, const void* blob,
                                        size_t len);
/* Advance several slabs of ONE process in lockstep (one step of each in turn),
 * the single-process analogue of MultiBlockRun::advance (multiblock.cpp:376-419).
 * Slabs on one device that move <= 64 MB per step replay one CUDA graph of
 * eight steps of every slab (DLB_GROUP_GRAPH=0/1 overrides): the call then
 * returns after enqueueing, as for single slabs. */
DLB_API dlb_status dlb_lattices_step(dlb_lattice** lats, size_t n, int64_t nsteps);

/* ---- GPU-resident diagnostics (the sampling step after the update) ----------
 * Replaces the host post-processing of Driver::sample / porous_extras
 * (runner.cpp:346-423) over gather_macroscopic (multiblock.cpp:443-484):
 * kinetic energy (diagnostics.cpp:25-31), FD8 vorticity + enstrophy (:33-120),
 * the cavity convergence sums (runner.cpp:433-444) and the porous plane / sample
 * means (runner.cpp:346-399), computed from the resident state.
 *
 * Every reduction reproduces diag::tree_sum (diagnostics.cpp:10-18) BIT FOR BIT:
 * the value sequence (x fastest, restricted / compacted as the runner builds
 * its vectors) is split by the same recursive halving; each slab reduces on the
 * device the maximal tree nodes that lie inside its segment of the global
 * sequence, and dlb_tree_combine evaluates the nodes above them on the host.
 * Leaves (<= 8 values, summed sequentially) cut by a segment boundary are
 * returned as raw values (len 0). */
typedef enum dlb_quantity {
    DLB_Q_KINETIC = 0,        /* 0.5*|u|^2, all cells */
    DLB_Q_ENSTROPHY = 1,      /* 0.5*|curl_fd8 u|^2, cells with a full stencil */
    DLB_Q_DU_NUM = 2,         /* |u - u_snapshot|^2, all cells */
    DLB_Q_DU_DEN = 3,         /* |u|^2, all cells */
    DLB_Q_PRESSURE_FLUID = 4, /* cs2*rho, fluid cells with x in [x_begin, x_end) */
    DLB_Q_UX_FLUID = 5,       /* ux, fluid cells with x in [x_begin, x_end) */
    DLB_Q_UX_ALL = 6,         /* ux, all cells with x in [x_begin, x_end) */
    DLB_Q_RHO_FLUID = 7,      /* rho, fluid cells with x in [x_begin, x_end) */
} dlb_quantity;

typedef struct dlb_reduce_args {
    int32_t quantity;     /* dlb_quantity */
    int32_t periodic[3];  /* ENSTROPHY: periodicity of the GLOBAL domain (valid-cell box) */
    int64_t x_begin;      /* masked quantities: x window */
    int64_t x_end;
    /* ENSTROPHY on a slab that does not hold the whole z extent: velocity of the
     * 4 global planes below z_origin / above z_origin + nz, host arrays laid out
     * [plane][ux|uy|uz][y][x] as dlb_lattice_velocity_planes returns them (NULL
     * where the stencil never reaches: non-periodic domain ends). */
    const double* halo_below;
    const double* halo_above;
} dlb_reduce_args;

/* One reduced node of the global tree: len >= 1 -> tree_sum of values
 * [lo, lo + len); len == 0 -> the raw value at index lo. */
typedef struct dlb_tree_part {
    int64_t lo;
    int64_t len;
    double value;
} dlb_tree_part;

/* Number of values this slab contributes to the quantity's sequence. */
DLB_API dlb_status dlb_lattice_reduce_count(dlb_lattice* lat, const dlb_reduce_args* args,
                                            int64_t* count_out);
/* Tree parts of this slab's segment [seg_begin, seg_begin + count) of a global
 * sequence of n_total values. parts may be NULL to query the number (n_out). */
DLB_API dlb_status dlb_lattice_reduce_parts(dlb_lattice* lat, const dlb_reduce_args* args,
                                            int64_t n_total, int64_t seg_begin,
                                            dlb_tree_part* parts, size_t cap, size_t* n_out);
/* One-slab convenience: count, parts and combine -> tree_sum of the sequence. */
DLB_API dlb_status dlb_lattice_reduce(dlb_lattice* lat, const dlb_reduce_args* args,
                                      double* sum_out, int64_t* count_out);
/* Host: tree_sum of a global sequence of n_total values from the parts of all
 * slabs (any order). DLB_ERROR_INVALID_ARGUMENT if a needed node is missing. */
DLB_API dlb_status dlb_tree_combine(int64_t n_total, const dlb_tree_part* parts, size_t n,
                                    double* sum_out);
/* Host: the parts segment [seg_begin, seg_end) of an n_total-value sequence
 * owns (values left 0) -- for callers that reduce their own segments. */
DLB_API dlb_status dlb_tree_plan(int64_t n_total, int64_t seg_begin, int64_t seg_end,
                                 dlb_tree_part* parts, size_t cap, size_t* n_out);
/* Host: diag::tree_sum (diagnostics.cpp:10-18) of a host array. */
DLB_API dlb_status dlb_tree_sum(const double* values, int64_t n, double* sum_out);
/* Fused collide + reduce (the paper's transform_reduce): the LAST
 * step of the next dlb_lattice_step call also writes the new state's per-cell
 * kinetic energy, so the following DLB_Q_KINETIC reduction reads 8 B/cell
 * instead of the populations (bit-identical values). *fused_out = 0 when the
 * lattice has no fused variant (fast arithmetic, AA, z-slab, regularized
 * fix-ups); the reduction then runs unfused. */
DLB_API dlb_status dlb_lattice_request_kinetic(dlb_lattice* lat, int32_t* fused_out);
/* Keep the current velocity field on the device as the DU_NUM reference
 * (the runner's prev_ux/uy/uz, runner.cpp:445-448). */
DLB_API dlb_status dlb_lattice_snapshot_velocity(dlb_lattice* lat);
/* Velocity of local planes [z0, z0 + nz) as [plane][ux|uy|uz][y][x] doubles
 * (gather_macroscopic semantics): the halo planes a neighbouring slab needs. */
DLB_API dlb_status dlb_lattice_velocity_planes(dlb_lattice* lat, int32_t z0, int32_t nz,
                                               double* out);

/* ---- drop-in for collide_and_stream<T> on a host AcceleratedBlock ----------- */
/* Envelope-inclusive SoA arrays exactly as AcceleratedBlock<T> holds them
 * (accelerated_lattice.hpp:86-112): f_in/f_out q*ext[0]*ext[1]*ext[2] values,
 * tag/param_index ext-volume int32. Pre: envelope of f_in current.
 * Post, f_out != NULL: the new interior state was written into the f_out
 * buffer, the previous state is left in the f_in
 * buffer, and the view's two pointers are SWAPPED -- view->f_in is the new
 * state, as after the reference's std::swap of the two arrays
 * (accelerated_lattice.cpp:199); callers owning the arrays swap them when the
 * pointers came back swapped. f_out == NULL: the new state
 * overwrites the interior of f_in in place (its envelope untouched).
 * f_out's envelope: pageable buffers -- untouched, as by the reference's
 * step_range (accelerated_lattice.cpp:126-153); pinned buffers (the copy-back
 * moves whole planes) -- the z envelope planes untouched, the x / y envelope
 * cells of the interior planes set to f_in's (identical whenever the two
 * buffers hold the same envelope: a bounded block's, or a periodic one the
 * caller refreshes before each step; DLB_BLOCK_D2H_ROWS=1 leaves them
 * untouched too, and costs 20-30 % of the end-to-end rate).
 * Errors (DLB_ERROR_DISPATCH ...) leave both buffers and the view unchanged. */
typedef struct dlb_block_view {
    int32_t precision_bits;
    int32_t q;
    int64_t interior[3];
    void* f_in;
    void* f_out;
    const int32_t* tag;
    const int32_t* param_index;
} dlb_block_view;
DLB_API dlb_status dlb_collide_and_stream(const dlb_registry* reg, dlb_block_view* block,
                                          const int32_t* dispatch_tags, size_t n_dispatch,
                                          int32_t nthreads);
/* refresh_envelope_periodic<T> (accelerated_lattice.hpp:130-132) on the same
 * host block: copy interior edge planes into the opposite envelope along the
 * periodic axes (x, then y over full x rows, then z over full planes). */
DLB_API dlb_status dlb_refresh_envelope_periodic(dlb_block_view* block, const int32_t* periodic);
/* The call keeps a device context per block shape (mirrors, slots, recipes)
 * for the next call on the same block; it is tied to the registry's content
 * (a new registration or dlb_registry_free invalidates it). Release them all
 * (device memory back) / query how many are held. */
DLB_API void dlb_block_cache_release(void);
DLB_API dlb_status dlb_block_cache_info(size_t* entries, int64_t* device_bytes);
/* Pinned host memory for the block API (page-locked, for full-rate copies). */
DLB_API dlb_status dlb_host_alloc(size_t bytes, void** out);
DLB_API void dlb_host_free(void* ptr);

/* ---- case input generators (src/cases.cpp) ------------------------------------ */
/* Random Boolean sphere pack written as the reference's raw 8-bit voxel format
 * (x fastest, 255 = solid; cases.cpp:86-111): spheres of radius r voxels with
 * uniform centres (mt19937_64 seed) are added, periodic placement, until the
 * porosity drops to target_porosity or below. */
DLB_API dlb_status dlb_case_sphere_pack(int64_t nx, int64_t ny, int64_t nz, double radius,
                                        double target_porosity, uint64_t seed, uint8_t* out,
                                        double* porosity_out);

#ifdef __cplusplus
}
#endif

#endif /* DLB_H */
