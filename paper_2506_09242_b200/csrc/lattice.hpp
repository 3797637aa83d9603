// Device lattice runtime: one z-slab of the domain resident in HBM.
//
// Mirrors the reference's AcceleratedBlock<T> + collide_and_stream<T> +
// MultiBlockRun<T> (proj/include/dolb/accelerated_lattice.hpp:86-127,
// proj/include/dolb/multiblock.hpp:119-176) with B200-native storage: padded
// SoA direction arrays with a one-cell envelope, u8 slot array, recipes in
// kernel parameter space, and a z-slab halo pushed over peer memory.
#pragma once

#include <cuda_runtime.h>

#include <array>
#include <cstdint>
#include <functional>
#include <memory>
#include <set>
#include <string>
#include <vector>

#include "../../include/dlb.h"
#include "chain.hpp"
#include "kernels.cuh"

namespace dlb {

void cuda_check(cudaError_t e, const char* what);

// Makes `dev` current for the scope of a Lattice entry point and restores the
// caller's device afterwards: slabs of one process may sit on different GPUs,
// and every launch / allocation must land on the slab's own device.
class DeviceGuard {
  public:
    explicit DeviceGuard(int dev) {
        if (cudaGetDevice(&prev_) != cudaSuccess) prev_ = -1;
        if (prev_ == dev) prev_ = -1;
        else cuda_check(cudaSetDevice(dev), "cudaSetDevice");
    }
    ~DeviceGuard() {
        if (prev_ >= 0) cudaSetDevice(prev_);
    }
    DeviceGuard(const DeviceGuard&) = delete;
    DeviceGuard& operator=(const DeviceGuard&) = delete;

  private:
    int prev_ = -1;
};

// Halo neighbour of a slab (the lower one at z = -1, the upper at z = nz).
struct Peer {
    bool linked = false;
    bool other_gpu = false;              // the neighbour's memory is on another GPU (NVLink / P2P)
    void* buf[2] = {nullptr, nullptr};   // peer populations, interior origin of direction 0
    long long dstride = 0;
    int nz = 0;
    unsigned long long* flag = nullptr;  // where to signal our progress in the peer's memory
    std::vector<void*> ipc_opened;       // bases opened through CUDA IPC (closed on free)
};

class Lattice {
  public:
    Lattice(const dlb_lattice_desc& desc, const DynamicsRegistry& reg);
    ~Lattice();
    Lattice(const Lattice&) = delete;
    Lattice& operator=(const Lattice&) = delete;

    void set_slots(const int32_t* slots);
    void set_uniform_slot(int32_t slot);
    void set_dispatch(const int32_t* tags, std::size_t n);
    void fill_equilibrium(const double* rho, const double* ux, const double* uy, const double* uz);
    void fill_uniform(double rho, double ux, double uy, double uz);
    void fill_tgv(int64_t L, double u_inf);
    void upload(const double* canon);
    void download(double* canon);
    void download_raw(void* canon);
    // Envelope-inclusive host block (AcceleratedBlock layout) in the storage type.
    void upload_block(const void* f, const int64_t ext[3]);
    void download_block_interior(void* f, const int64_t ext[3], int which);
    // One step of a caller-owned, page-locked AcceleratedBlock (envelope
    // included, refreshed by the caller), pipelined over z-chunks: host->device
    // copies of the next chunk, the step of this chunk and device->host copies
    // of the previous one run concurrently (both PCIe directions busy).
    // f_out (may be null): the new state goes into f_out instead of back into f_in
    void step_host_block(void* f_in, const int64_t ext[3], void* f_out = nullptr);
    // The same in two halves: begin enqueues every H2D chunk and its compute
    // (device-side writes only), finish enqueues the copy-back into the
    // caller's block; abort drops a begun step. Lets the caller's eager
    // dispatch scan overlap the transfers while still failing before any write.
    void begin_host_block(void* f_in, const int64_t ext[3], void* f_out = nullptr);
    // gate(z_end), when given, is asked before the copy-back of the chunk that
    // ends at interior plane z_end: -1 when the slots of planes [0, z_end) are
    // confirmed, else the first plane whose slots changed -- then the pipeline
    // drains, reslot() installs the new slots, and the chunks from that one on
    // are recomputed (the input mirror still holds the whole input state).
    void finish_host_block(const std::function<int(int)>& gate = {}, const std::function<void()>& reslot = {});
    void abort_host_block();
    void step(int64_t nsteps);
    void enqueue_step();  // one step, no dispatch check (group stepping)
    // Several slabs of one process in lockstep (MultiBlockRun::advance,
    // multiblock.cpp:376-419): long runs replay one CUDA graph holding eight
    // steps of every slab (slabs on one device), so the host does not enqueue
    // ~5 operations per slab and step. Dispatch is checked by the caller.
    static void step_group(const std::vector<Lattice*>& lats, int64_t nsteps);
    void check_dispatch() const;
    void synchronize();
    void checksum(unsigned long long* per_dir, bool active_only = false);
    void gather_macroscopic(double* rho, double* ux, double* uy, double* uz);  // q order-independent 64-bit sums
    double time_steps(int64_t nsteps);

    // Halo wait limit per step (a neighbour that does not finish its boundary
    // planes within it makes the step fail with DLB_ERROR_EXCHANGE).
    void set_halo_timeout(double seconds);
    // 0 = not linked, 1 = linked to a slab on the same GPU, 2 = on another GPU;
    // halo_bytes = bytes this slab pushes to its neighbours per step
    void links(int* lower, int* upper, int64_t* halo_bytes) const;
    // DLB_TRACE_HALO timeline of the linked steps since the last call (ms from
    // the first event; 5 per step: halo wait begin / end, boundary end on the
    // halo stream, interior begin / end on the main stream)
    std::vector<double> halo_trace(bool consume = true);
    void link_lower(Lattice& lower);  // same process
    void exchange();                  // prime the neighbours' ghost planes (clears an exchange error)
    void quiesce();                   // wait for this slab's streams (no error check)
    std::vector<uint8_t> export_ipc() const;
    void link_ipc(int side, const void* blob, std::size_t len);

    cudaStream_t stream() const { return stream_; }
    int64_t steps_done() const { return steps_; }
    int64_t bytes_per_cell() const;
    int64_t step_bytes() const;
    int64_t device_bytes() const { return device_bytes_; }
    int launches_per_step() const;
    const char* kernel_name() const {
        if (kernel_tma_ && !(lower_.linked || upper_.linked)) return kernel_tma_->name;
        if (kernel_cmp_ && !(lower_.linked || upper_.linked)) return kernel_cmp_->name;
        if (kernel_vec_ && !(lower_.linked || upper_.linked)) return kernel_vec_->name;
        if (kernel_segbb_ && !(lower_.linked || upper_.linked)) return kernel_segbb_->name;
        if (kernel_seg_ && !(lower_.linked || upper_.linked)) return kernel_seg_->name;
        if (kernel_main_ && !fixups_.empty() && !(lower_.linked || upper_.linked)) return kernel_main_->name;
        return kernel_ ? kernel_->name : "<none>";
    }
    int slab_planes() const { return d_.dims[2]; }
    int64_t cells() const { return int64_t(d_.dims[0]) * d_.dims[1] * d_.dims[2]; }
    int bits() const { return d_.precision_bits; }
    int q() const { return d_.q; }
    void set_periodic_override(bool x, bool y, bool z);

    // GPU-resident diagnostics (diag.cu): split deterministic tree reductions
    // of per-cell quantities of the current state (include/dlb.h).
    int64_t reduce_count(const dlb_reduce_args& a) const;
    void reduce_parts(const dlb_reduce_args& a, int64_t n_total, int64_t seg_begin,
                      std::vector<dlb_tree_part>& out);
    void snapshot_velocity();
    // The next step also writes the new state's per-cell kinetic energy (one
    // 8-B store per cell in the collide-stream kernel), so the following
    // DLB_Q_KINETIC reduction reads 8 B/cell instead of the populations.
    // Returns false when this lattice has no fused variant (reduction unfused).
    bool request_kinetic();
    bool kinetic_fused_current() const { return d_ke_ && ke_step_ == steps_; }
    void velocity_planes(int z0, int nz, double* out);

  private:
    void select_kernel();
    template <typename T>
    void launch_step(int parity);
    void copy_canonical(void* host, bool to_device, bool as_double, int elem_bytes);
    void* origin(int which) const;  // interior origin of direction 0 of buffer `which`
    bool split() const { return d_.global_nz != d_.dims[2]; }
    bool aa() const { return d_.layout == DLB_LAYOUT_AA; }
    // layout of the current state for fills / canonical access (canon_load's aa_mode)
    int aa_fill_mode() const { return !aa() ? 0 : (aa_odd_layout_ ? 2 : 1); }
    void reset_aa();
    void check_error_flag();

    dlb_lattice_desc d_;
    int device_ = 0;
    cudaStream_t stream_ = nullptr;
    cudaEvent_t ev0_ = nullptr, ev1_ = nullptr;
    // linked slabs: halo wait + boundary launch on halo_stream_ (high priority)
    // concurrent with the interior launch on stream_, forked / joined per step
    cudaStream_t halo_stream_ = nullptr;
    cudaEvent_t ev_fork_ = nullptr, ev_join_ = nullptr;
    cudaEvent_t ev_wait_ = nullptr;       // AA: the interior launch starts after the halo wait
    unsigned long long halo_timeout_ns_ = 20ull * 1000 * 1000 * 1000;  // DLB_HALO_TIMEOUT_MS / set_halo_timeout
    bool trace_halo_ = false;             // DLB_TRACE_HALO
    bool exchange_failed_ = false;        // a timed-out halo wait was reported (cleared by exchange)
    bool overlap_ = true;                 // DLB_HALO_OVERLAP (0: serialised halo + interior)
    std::vector<cudaEvent_t> trace_ev_;   // 5 per linked step: wait0, wait1, boundary1, interior0, interior1
    Geo geo_{};
    int align_ = 32;            // elements per 128 B
    int skip_group_ = 8;        // masked porous sweep: cells per skip group (power of two <= 32)
    int64_t masked_cells_ = -1; // masked porous sweep: cells in non-skipped groups (-1: not masked)
    // compacted masked sweep (single slab): listed segment indices and kernel
    unsigned* d_seg_ = nullptr;
    long long nseg_ = 0;
    const KernelEntry* kernel_seg_ = nullptr;
    bool seg_fused_reg_ = false;  // k_seg runs the regularized cells itself (no fix-up launches)
    int pull_threads_ = 128;      // dense / AA sweep threads per block (DLB_PULL_THREADS)
    int seg_prefetch_ = 74;       // segment-entry L2 prefetch distance in blocks (DLB_SEG_PREFETCH)
    int seg_block_ = 256;         // segment sweep threads per block (DLB_SEG_BLOCK)
    int seg_pack_ = 0;            // k_seg entry packing (bs | by << 8), 0 = linear segment index
    bool dense_seg_ = false;      // dense porous sweep as k_seg over every segment (fp64 with regularized planes)
    // fluid-segment sweep (k_segbb): segments with a collision cell, their
    // per-cell bounce-back link masks, the wall cells finalized lazily
    unsigned* d_fseg_ = nullptr;
    unsigned* d_flink_ = nullptr;
    unsigned long long* d_bbfin_ = nullptr;
    long long nfseg_ = 0, nbbfin_ = 0, fseg_cells_ = 0;
    const KernelEntry* kernel_segbb_ = nullptr;
    bool bb_prologue_ = true;  // next step must be a full k_seg step (buffers not yet ping-pong current)
    bool bb_dirty_ = false;    // wall cells outside the fluid segments are behind the state
    void build_fluid_segments(const std::vector<uint8_t>& u8);
    void finalize_walls();
    // compacted porous sweep (k_cmp, porous_compact.cu): listed segments and the
    // segments they pull from, gathered into row-major compact arrays
    void* cbuf_[2] = {nullptr, nullptr};
    long long cstride_ = 0;                        // elements per compact direction array
    long long ncomp_ = 0, ncl_ = 0, ncfix_ = 0;    // compact segments, listed segments, fix-up cells
    int cgshift_ = 0;
    unsigned* d_cseg_ = nullptr;    // listed segment -> compact index | valid lanes << 26
    unsigned* d_crows_ = nullptr;   // [8][ncl_] compact index of the same-x segment in the neighbouring rows
    long long* d_coff_ = nullptr;   // compact segment -> dense offset of its first cell
    int* d_cx0_ = nullptr;          // compact segment -> x of its first cell
    uint8_t* d_cslot_ = nullptr;    // per compact cell
    unsigned* d_cfix_ = nullptr;    // regularized cells (listed segment << gshift | lane)
    const KernelEntry* kernel_vec_ = nullptr;  // 128-bit vectorised dense sweep (DLB_VEC=1)
    const KernelEntry* kernel_cmp_ = nullptr;
    const KernelEntry* kernel_cmp_fix_ = nullptr;
    bool cmp_valid_ = false;        // the compact arrays hold the current state
    bool cmp_dirty_ = false;        // the dense layout is behind them
    int64_t cmp_bytes_ = 0;
    void build_compact(const std::vector<uint8_t>& u8, const std::vector<uint8_t>& nodyn);
    void free_compact();
    void prepare_compact();   // gather before the first compact step after a state write
    void scatter_compact();   // dense layout up to date (before reads)
    // fused kinetic energy (KM_KE variant): per-cell values of the state after
    // step ke_step_, consumed by the next DLB_Q_KINETIC reduction
    const KernelEntry* kernel_ke_ = nullptr;
    // persistent cooperative multi-step sweep for small lattices (k_pull_coop)
    const KernelEntry* kernel_coop_ = nullptr;
    int coop_grid_ = 0;
    template <typename T>
    void launch_coop(int64_t nsteps);
    double* d_ke_ = nullptr;
    bool ke_requested_ = false;
    int64_t ke_step_ = -1;
    long long base_off_ = 0;    // elements from array start to the interior origin
    void* buf_[2] = {nullptr, nullptr};
    int cur_ = 0;               // buffer holding the current state (f_in)
    uint8_t* d_slot_ = nullptr;
    int uniform_slot_ = -1;
    bool slots_set_ = false;
    std::vector<int32_t> present_slots_;
    bool untagged_ = false;
    std::set<int> dispatch_;
    bool dispatch_set_ = false;
    // snapshot of the registry (MultiBlockRun compiles recipes at construction,
    // multiblock.cpp:419)
    std::vector<DynamicsChain> chains_;
    std::vector<int> tag_of_slot_;
    std::vector<std::string> tag_names_;
    unsigned km_needed_ = 0;
    bool xrec_ = false;          // more instances than the parameter-space table: KM_XREC kernels
    void* d_xrec_ = nullptr;     // DevRecipe<T>[instances] in global memory (xrec_)
    const KernelEntry* kernel_ = nullptr;
    const KernelEntry* kernel_odd_ = nullptr;  // AA: odd-step kernel (kernel_ is the even one)
    const KernelEntry* kernel_link_ = nullptr;      // AA linked slabs: boundary-plane even / odd kernels
    const KernelEntry* kernel_odd_link_ = nullptr;
    bool aa_odd_layout_ = true;                // AA: state is in the odd / upload layout
    // halo
    Peer lower_, upper_;
    unsigned long long* d_flags_ = nullptr;  // [0] from lower, [1] from upper, [2] my step, [3] error
    unsigned int* d_counter_ = nullptr;      // last-block ticket of the boundary launch
    int64_t steps_ = 0;
    int64_t halo_steps_ = 0;  // linked steps enqueued (host mirror of flags[2] once they ran)
    int64_t device_bytes_ = 0;
    void* staging_ = nullptr;
    std::size_t staging_bytes_ = 0;
    // sparse porous mode (DLB_FLAG_SKIP_NODYNAMICS on a single slab): per-slot
    // row-major lists of the cells that move populations, one launch each
    struct ListLaunch {
        int slot;
        long long offset, count;
        const KernelEntry* kernel;
    };
    bool sparse_ = false;
    // rare-kind split (two-population, unlinked): the dense sweep runs without
    // the regularized boundary code (fewer registers, higher occupancy) and
    // list launches recompute the regularized cells afterwards
    std::vector<ListLaunch> fixups_;
    unsigned long long* d_fix_ = nullptr;
    const KernelEntry* kernel_main_ = nullptr;
    void build_fixups(const std::vector<uint8_t>& u8);
    std::vector<ListLaunch> lists_;
    unsigned long long* d_list_ = nullptr;
    int64_t step_bytes_ = 0;  // algorithmic bytes per step
    void build_lists(const std::vector<uint8_t>& u8);
    void check_skip_precondition(const std::vector<uint8_t>& u8, const std::vector<uint8_t>& nodyn) const;
    // TMA-staged dense kernel (single slab): tensor maps of both buffers, and
    // whether the input buffer's envelope holds the periodic images
    const KernelEntry* kernel_tma_ = nullptr;
    CUtensorMap tmap_[6];            // [0..1] box maps (k_tma), [2..3] row maps (k_tmarow), [4..5] k_tmablk
    bool blk_ok_ = false;
    bool row_ok_ = false;
    int row_nb_ = 0, row_bw_ = 0;    // k_tmarow: boxes per tile and box width (elements)
    int row_tw_ = 0;                 // k_tmarow: cells per work unit (a row or an x-split of it)
    CUtensorMap* d_tmap_ = nullptr;  // the two maps in device global memory
    int tma_xoff_ = 0;
    bool tma_ok_ = false;
    bool envelope_valid_ = false;
    int tma_grid_ = 0;
    void setup_tma();
    void refresh_envelope(int which);
    template <typename T>
    void launch_tma(StepArgs<T>& a, int parity);
    // CUDA graph of two consecutive steps (parity 0 -> 1 -> 0), replayed by
    // step() / time_steps(); invalidated whenever kernels, slots or links change
    cudaGraphExec_t graph_ = nullptr;
    uint64_t graph_version_ = 0;  // changes whenever the captured work would change (group graph cache key)
    void invalidate_graph();
    void ensure_graph();
    // host-block (zero-copy) path
    void* blk_out_ = nullptr;
    std::size_t blk_out_bytes_ = 0;
    cudaStream_t copy_stream_ = nullptr;
    cudaStream_t h2d_stream_ = nullptr;
    std::vector<cudaEvent_t> blk_ev_;
    cudaEvent_t blk_tr_[5] = {nullptr, nullptr, nullptr, nullptr, nullptr};  // DLB_TRACE_BLOCK timeline
    struct BlockPlan {
        void* f_in = nullptr;
        void* f_out = nullptr;  // where the new state goes (f_in when in place)
        void* din = nullptr;
        void* dout = nullptr;
        long long vol = 0;
        int plane = 0, nz = 0, zc = 1, nchunks = 0, elem = 4;
        int pitch = 0, nx = 0, ny = 0;  // host row pitch (x extent + envelope), interior x / y
        int issued = 0;         // chunks whose H2D + compute are enqueued
        int ahead = 2;          // H2D chunks allowed ahead of the D2H copy-back (DLB_BLOCK_AHEAD, 0 = all)
        unsigned gx = 1, gy = 1, bx = 32, by = 8;
        int loaded = 0;         // host planes [0, loaded) on the device
        int copied = 0;         // chunks whose copy-back is enqueued
        bool pending = false;
    } blk_;
    std::vector<uint8_t> blk_args_;  // the StepArgs<T> of the pending block step
    void issue_block_chunk(int c);
    template <typename T>
    void refill_block_recipes();
    void block_copy(cudaStream_t st, void* host, void* dev, bool up, int p0, int p1);
    void block_copy_back_interior(cudaStream_t st, int p0, int p1);
    template <typename T>
    void fill_recipes(StepArgs<T>& a) const;
    template <typename T>
    void launch_host_block(void* f_in, const int64_t ext[3], void* f_out);
    // diagnostics state (diag.cu)
    double* d_uprev_ = nullptr;  // velocity snapshot [ux | uy | uz] x cells
    void* diag_buf_ = nullptr;
    std::size_t diag_bytes_ = 0;
    void* diag_scratch(std::size_t min_bytes);
    template <typename T>
    void diag_impl(const dlb_reduce_args& a, int64_t n_total, int64_t seg_begin,
                   std::vector<dlb_tree_part>& out);
    template <typename T>
    void velocity_planes_impl(int z0, int nz, double* dev_out);
    void* diag_slots();  // per-slot kind / fluid flag / wall velocity on the device
};

// Sphere-pack porous medium generator (cases.cpp raw voxel format).
double sphere_pack(int64_t nx, int64_t ny, int64_t nz, double radius, double target_porosity,
                   uint64_t seed, uint8_t* out);

}  // namespace dlb
