// Launch-side description of the collide-and-stream kernels, shared by the
// kernel translation units (compiled once per arithmetic mode) and the host.
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>

#include "lbm_cell.cuh"

namespace dlb {

// Recipes of the first kMaxSlots registry instances travel in kernel
// parameter space (constant bank); larger registries (up to kMaxInstances,
// the u8 slot array's range) use the KM_XREC kernels, which read the whole
// table from global memory.
constexpr int kMaxSlots = 16;
constexpr int kMaxInstances = 256;

// Device layout of one direction array (SoA, envelope-inclusive):
//   element (x, y, z) of direction i, with x in [-1, nx], y in [-1, ny],
//   z in [-1, nz] (the -1 / n layers are the envelope / ghost planes), sits at
//   base_i + z*plane + y*pitch + x, where base_i points at interior (0,0,0).
//   pitch >= nx + 2 is a multiple of 128 B, and base_i is 128 B aligned, so
//   every interior row starts on a cache line; x = -1 lives in the previous
//   row's padding.
struct Geo {
    int nx, ny, nz;
    int pitch;        // elements per row
    int plane;        // pitch * (ny + 2)
    int per_x, per_y, per_z;  // wrap in-kernel along this axis (else read the envelope)
    long long dstride;        // elements per direction array
};

constexpr int kMaxQ = 27;

template <typename T>
struct StepArgs {
    // per-direction interior origins (host-computed: keeps the 64-bit
    // direction offsets out of the per-thread address arithmetic)
    const T* fin[kMaxQ];
    T* fout[kMaxQ];
    const uint8_t* slot;    // nx*ny*nz registry slots (x fastest) or nullptr if uniform
    int uniform_slot;
    int z_begin, z_step;    // plane z = z_begin + blockIdx.z * z_step
    // masked porous sweep (KM_SKIP): x-aligned groups of skip_group cells (a
    // power of two <= 32, one 32-B or 64-B memory segment) are skipped only
    // when every cell of the group is NoDynamics
    int skip_group;
    Geo g;
    // z-slab halo push over peer memory (nullptr when absent): after the
    // collision, cells of the top plane store their c_z = +1 populations into
    // the upper neighbour's ghost plane z = -1, cells of the bottom plane their
    // c_z = -1 populations into the lower neighbour's ghost plane z = nz_lower.
    T* push_up;
    T* push_down;
    long long up_dstride, down_dstride;
    int down_ghost_z;
    // Completion signal of the boundary launch (nullptr otherwise): every
    // block fences its peer stores, the last block (ticket == gridsize - 1)
    // increments *my_step and release-stores it into both neighbours' flags.
    unsigned int* counter;
    unsigned long long* my_step;
    unsigned long long* sig_up;
    unsigned long long* sig_down;
    DevRecipe<T> rec[kMaxSlots];
    // KM_KE variant: per-cell kinetic energy of the new state, x fastest
    // (appended last so the other kernels' parameter offsets do not move)
    double* ke;
    // linked slabs: the exchange error flag (flags[3]); a launch that finds it
    // set writes nothing (a timed-out halo wait fails the step and every later
    // one, so the last completed state stays intact)
    const unsigned long long* err;
    // KM_XREC kernels: the full recipe table (any registry size) in global memory
    const DevRecipe<T>* xrec;
};

// Compacted porous sweep (k_cmp): the populations of the listed skip segments
// (and of the never-updated segments they pull from) stored contiguously in
// row-major segment order, G = 1 << gshift cells per segment. Segment m's cell
// `lane` of direction i sits at fin[i][m * G + lane]; because the order is
// row-major, the x-neighbour segments of a source segment are m - 1 / m + 1.
struct CmpArgs {
    const unsigned* seg;    // per listed segment: compact index | (valid lanes << 26)
    const unsigned* rows;   // [8][nlist]: compact index of the same-x segment in row (y + dy, z + dz)
    const uint8_t* slot;    // per compact cell: registry slot
    const unsigned* fix;    // k_cmp FIX variant: listed cells (listed segment << gshift | lane)
    long long n;            // threads (cells) of the launch
    long long nlist;        // listed segments
    int gshift;
};

// Row-table index of the row offset (dy, dz) != (0, 0).
__host__ __device__ constexpr int cmp_row(int dy, int dz) {
    return (dz + 1) * 3 + (dy + 1) - (((dz + 1) * 3 + (dy + 1)) > 4 ? 1 : 0);
}

// Recipe of slot s as the instantiation reads it.
template <unsigned KM, typename T>
__device__ __forceinline__ const DevRecipe<T>& recipe_of(const StepArgs<T>& a, int s) {
    if constexpr ((KM & KM_XREC) != 0) return a.xrec[s];
    else return a.rec[s];
}

// kernel families: dense two-population, AA even / odd, sparse lists (fluid / masked walls)
enum Layout : int { LAYOUT_TWO_POP = 0, LAYOUT_AA = 1, LAYOUT_AA_ODD = 2, LAYOUT_LIST = 3, LAYOUT_LIST_MASKED = 4,
                    LAYOUT_TMA = 5, LAYOUT_SEG = 6, LAYOUT_TMAROW = 7,
                    LAYOUT_COOP = 8, LAYOUT_TMABLK = 9, LAYOUT_SEGBB = 10,
                    LAYOUT_AA_LINK = 11, LAYOUT_AA_ODD_LINK = 12, LAYOUT_CMP = 13, LAYOUT_CMP_FIX = 14,
                    LAYOUT_VEC = 15 };

struct KernelEntry {
    int precision_bits;
    int q;
    unsigned km;
    int layout;
    const void* fn;  // __global__ function pointer
    const char* name;
    int tile_x = 0, tile_y = 0, stages = 0;  // TMA kernels: tile shape and ring depth
    int cpt = 1;                             // segment kernels: cells per thread
    int warps = 0;                           // row-staged TMA kernels: consumer warps per CTA
    int minb = 0;                            // k_pull tuning entries: occupancy target override
};

// Kernel tables of the two arithmetic modes (one translation unit each).
namespace exact { const KernelEntry* kernel_table(int* n); }
namespace fast { const KernelEntry* kernel_table(int* n); }
// Lazy wall-cell update of the fluid-segment sweep (k_bb_finalize); cur / prev
// are the interior origins of direction 0 of the two buffers.
namespace exact {
void launch_bb_finalize(int bits, int q, void* cur, const void* prev, const Geo& g,
                        const unsigned long long* list, long long n, cudaStream_t st);
}

}  // namespace dlb
