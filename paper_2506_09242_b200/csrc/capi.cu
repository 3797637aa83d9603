// extern "C" boundary of libdlb_b200.so (include/dlb.h). Exceptions map to
// status codes the way the reference's C interface does (proj/src/capi.cpp:20-39);
// the message goes to a thread-local last-error buffer (capi.cpp:13-18).
#include <chrono>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <functional>
#include <atomic>
#include <map>
#include <memory>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include "../../include/dlb.h"
#include "chain.hpp"
#include "lattice.hpp"
#include "tree.hpp"

struct dlb_registry {
    dlb::DynamicsRegistry reg;
    // identity of this registry's content for the host-block device cache:
    // a process-unique serial, and a generation bumped by every registration
    uint64_t serial = 0;
    uint64_t generation = 0;
};

struct dlb_lattice {
    std::unique_ptr<dlb::Lattice> lat;
};

namespace {

thread_local std::string g_last_error;

dlb_status fail(dlb_status s, const std::string& msg) {
    g_last_error = msg;
    return s;
}

template <typename Fn>
dlb_status guarded(Fn&& fn) {
    try {
        fn();
        return DLB_OK;
    } catch (const dlb::DispatchError& e) {
        return fail(DLB_ERROR_DISPATCH, e.what());
    } catch (const dlb::ExchangeError& e) {
        return fail(DLB_ERROR_EXCHANGE, e.what());
    } catch (const dlb::DeviceError& e) {
        return fail(DLB_ERROR_INTERNAL, e.what());
    } catch (const std::invalid_argument& e) {
        return fail(DLB_ERROR_CONFIG, e.what());
    } catch (const std::out_of_range& e) {
        return fail(DLB_ERROR_CONFIG, e.what());
    } catch (const std::domain_error& e) {
        return fail(DLB_ERROR_CONFIG, e.what());
    } catch (const std::runtime_error& e) {
        return fail(DLB_ERROR_IO, e.what());
    } catch (const std::exception& e) {
        return fail(DLB_ERROR_INTERNAL, e.what());
    } catch (...) {
        return fail(DLB_ERROR_INTERNAL, "unknown error");
    }
}

#define DLB_REQUIRE(cond)                                                          \
    do {                                                                           \
        if (!(cond)) return fail(DLB_ERROR_INVALID_ARGUMENT, "null argument: " #cond); \
    } while (0)

void write_string(const std::string& s, char* buf, size_t cap, size_t* len_out) {
    if (len_out) *len_out = s.size() + 1;
    if (buf == nullptr) return;  // size query
    if (cap < s.size() + 1) throw std::invalid_argument("buffer too small");
    std::memcpy(buf, s.c_str(), s.size() + 1);
}

// Cached device lattice for the host-block drop-in (one per block shape),
// valid for one registry content (serial + generation): a freed registry or a
// new registration never reuses stale recipes. Released by dlb_registry_free
// (its entries) and dlb_block_cache_release (all).
struct BlockCtx {
    std::unique_ptr<dlb::Lattice> lat;
    uint64_t reg_serial = 0, reg_generation = 0;
    std::vector<int32_t> slots;
    // per (y, z) row: the row's slot when all nx cells share it, else
    // kMixedRow -- the scan compares such rows against one value instead of
    // re-reading the cached slots (a third of the scan's host reads)
    std::vector<int64_t> row_slot;
};
constexpr int64_t kMixedRow = INT64_MIN;
std::mutex g_block_mu;
std::map<std::vector<int64_t>, BlockCtx> g_blocks;
std::atomic<uint64_t> g_registry_serial{0};

}  // namespace

extern "C" {

DLB_API const char* dlb_version(void) { return "dlb-b200 0.1 (sm_100a)"; }
DLB_API const char* dlb_last_error(void) { return g_last_error.c_str(); }

DLB_API dlb_status dlb_chain_canonical(const char* chain, char* buf, size_t cap, size_t* len_out) {
    DLB_REQUIRE(chain);
    return guarded([&] {
        const auto links = dlb::parse_chain_string(chain);
        dlb::validate_chain(links);
        write_string(dlb::chain_string(links), buf, cap, len_out);
    });
}

DLB_API dlb_status dlb_registry_new(dlb_registry** out) {
    DLB_REQUIRE(out);
    return guarded([&] {
        auto* r = new dlb_registry();
        r->serial = ++g_registry_serial;
        *out = r;
    });
}

DLB_API void dlb_registry_free(dlb_registry* reg) {
    if (!reg) return;
    {
        std::lock_guard<std::mutex> lock(g_block_mu);
        for (auto it = g_blocks.begin(); it != g_blocks.end();)
            it = it->second.reg_serial == reg->serial ? g_blocks.erase(it) : std::next(it);
    }
    delete reg;
}

DLB_API void dlb_block_cache_release(void) {
    std::lock_guard<std::mutex> lock(g_block_mu);
    g_blocks.clear();
}

DLB_API dlb_status dlb_block_cache_info(size_t* entries, int64_t* device_bytes) {
    DLB_REQUIRE(entries);
    std::lock_guard<std::mutex> lock(g_block_mu);
    *entries = g_blocks.size();
    if (device_bytes) {
        int64_t b = 0;
        for (const auto& kv : g_blocks)
            if (kv.second.lat) b += kv.second.lat->device_bytes();
        *device_bytes = b;
    }
    return DLB_OK;
}

DLB_API dlb_status dlb_registry_register(dlb_registry* reg, const char* chain, const double* params,
                                         size_t n_params, int32_t* slot_out) {
    DLB_REQUIRE(reg);
    DLB_REQUIRE(chain);
    DLB_REQUIRE(slot_out);
    DLB_REQUIRE(params || n_params == 0);
    return guarded([&] {
        dlb::DynamicsChain c;
        c.links = dlb::parse_chain_string(chain);
        dlb::validate_chain(c.links);
        c.params = dlb::deserialize_params(c.links, params, n_params);
        *slot_out = reg->reg.register_chain(c);
        ++reg->generation;
    });
}

DLB_API dlb_status dlb_registry_tag_for(const dlb_registry* reg, const char* chain, int32_t* tag_out) {
    DLB_REQUIRE(reg);
    DLB_REQUIRE(chain);
    DLB_REQUIRE(tag_out);
    return guarded([&] { *tag_out = reg->reg.tag_for(chain); });
}

DLB_API dlb_status dlb_registry_chain_for(const dlb_registry* reg, int32_t tag, char* buf, size_t cap,
                                          size_t* len_out) {
    DLB_REQUIRE(reg);
    return guarded([&] { write_string(reg->reg.chain_for(tag), buf, cap, len_out); });
}

DLB_API dlb_status dlb_registry_tag_of_slot(const dlb_registry* reg, int32_t slot, int32_t* tag_out) {
    DLB_REQUIRE(reg);
    DLB_REQUIRE(tag_out);
    return guarded([&] { *tag_out = reg->reg.tag_of_slot(slot); });
}

DLB_API dlb_status dlb_registry_counts(const dlb_registry* reg, int32_t* num_tags, int32_t* num_instances) {
    DLB_REQUIRE(reg);
    return guarded([&] {
        if (num_tags) *num_tags = reg->reg.num_tags();
        if (num_instances) *num_instances = reg->reg.num_instances();
    });
}

DLB_API dlb_status dlb_registry_slot_params(const dlb_registry* reg, int32_t slot, double* buf,
                                            size_t cap, size_t* len_out) {
    DLB_REQUIRE(reg);
    return guarded([&] {
        const auto& in = reg->reg.instance(slot);
        if (len_out) *len_out = size_t(in.param_len);
        if (!buf) return;
        if (cap < size_t(in.param_len)) throw std::invalid_argument("buffer too small");
        for (int64_t k = 0; k < in.param_len; ++k)
            buf[k] = reg->reg.params_table()[size_t(in.param_offset + k)];
    });
}

DLB_API dlb_status dlb_lattice_create(const dlb_lattice_desc* desc, const dlb_registry* reg,
                                      dlb_lattice** out) {
    DLB_REQUIRE(desc);
    DLB_REQUIRE(reg);
    DLB_REQUIRE(out);
    return guarded([&] {
        auto h = std::make_unique<dlb_lattice>();
        h->lat = std::make_unique<dlb::Lattice>(*desc, reg->reg);
        *out = h.release();
    });
}

DLB_API void dlb_lattice_free(dlb_lattice* lat) { delete lat; }

DLB_API dlb_status dlb_lattice_set_slots(dlb_lattice* lat, const int32_t* slots) {
    DLB_REQUIRE(lat);
    DLB_REQUIRE(slots);
    return guarded([&] { lat->lat->set_slots(slots); });
}

DLB_API dlb_status dlb_lattice_set_uniform_slot(dlb_lattice* lat, int32_t slot) {
    DLB_REQUIRE(lat);
    return guarded([&] { lat->lat->set_uniform_slot(slot); });
}

DLB_API dlb_status dlb_lattice_set_dispatch(dlb_lattice* lat, const int32_t* tags, size_t n) {
    DLB_REQUIRE(lat);
    DLB_REQUIRE(tags || n == 0);
    return guarded([&] { lat->lat->set_dispatch(tags, n); });
}

DLB_API dlb_status dlb_lattice_fill_equilibrium(dlb_lattice* lat, const double* rho, const double* ux,
                                                const double* uy, const double* uz) {
    DLB_REQUIRE(lat);
    DLB_REQUIRE(rho && ux && uy && uz);
    return guarded([&] { lat->lat->fill_equilibrium(rho, ux, uy, uz); });
}

DLB_API dlb_status dlb_lattice_fill_tgv(dlb_lattice* lat, int64_t L, double u_inf) {
    DLB_REQUIRE(lat);
    return guarded([&] { lat->lat->fill_tgv(L, u_inf); });
}

DLB_API dlb_status dlb_lattice_upload_populations(dlb_lattice* lat, const double* canon) {
    DLB_REQUIRE(lat);
    DLB_REQUIRE(canon);
    return guarded([&] { lat->lat->upload(canon); });
}

DLB_API dlb_status dlb_lattice_download_populations(dlb_lattice* lat, double* canon) {
    DLB_REQUIRE(lat);
    DLB_REQUIRE(canon);
    return guarded([&] {
        lat->lat->synchronize();
        lat->lat->download(canon);
    });
}

DLB_API dlb_status dlb_lattice_download_raw(dlb_lattice* lat, void* canon) {
    DLB_REQUIRE(lat);
    DLB_REQUIRE(canon);
    return guarded([&] {
        lat->lat->synchronize();
        lat->lat->download_raw(canon);
    });
}

DLB_API dlb_status dlb_lattice_step(dlb_lattice* lat, int64_t nsteps) {
    DLB_REQUIRE(lat);
    return guarded([&] { lat->lat->step(nsteps); });
}

DLB_API dlb_status dlb_lattice_synchronize(dlb_lattice* lat) {
    DLB_REQUIRE(lat);
    return guarded([&] { lat->lat->synchronize(); });
}

DLB_API dlb_status dlb_lattice_stream(dlb_lattice* lat, void** stream_out) {
    DLB_REQUIRE(lat);
    DLB_REQUIRE(stream_out);
    *stream_out = static_cast<void*>(lat->lat->stream());
    return DLB_OK;
}

DLB_API dlb_status dlb_lattice_steps_done(dlb_lattice* lat, int64_t* steps_out) {
    DLB_REQUIRE(lat);
    DLB_REQUIRE(steps_out);
    *steps_out = lat->lat->steps_done();
    return DLB_OK;
}

DLB_API dlb_status dlb_lattice_traffic(dlb_lattice* lat, int64_t* bytes_per_cell, int64_t* device_bytes,
                                       int32_t* launches_per_step) {
    DLB_REQUIRE(lat);
    if (bytes_per_cell) *bytes_per_cell = lat->lat->bytes_per_cell();
    if (device_bytes) *device_bytes = lat->lat->device_bytes();
    if (launches_per_step) *launches_per_step = lat->lat->launches_per_step();
    return DLB_OK;
}

DLB_API dlb_status dlb_lattice_gather_macroscopic(dlb_lattice* lat, double* rho, double* ux,
                                                  double* uy, double* uz) {
    DLB_REQUIRE(lat);
    DLB_REQUIRE(rho && ux && uy && uz);
    return guarded([&] { lat->lat->gather_macroscopic(rho, ux, uy, uz); });
}

DLB_API dlb_status dlb_lattice_reduce_count(dlb_lattice* lat, const dlb_reduce_args* args,
                                            int64_t* count_out) {
    DLB_REQUIRE(lat);
    DLB_REQUIRE(args && count_out);
    return guarded([&] { *count_out = lat->lat->reduce_count(*args); });
}

DLB_API dlb_status dlb_lattice_reduce_parts(dlb_lattice* lat, const dlb_reduce_args* args,
                                            int64_t n_total, int64_t seg_begin,
                                            dlb_tree_part* parts, size_t cap, size_t* n_out) {
    DLB_REQUIRE(lat);
    DLB_REQUIRE(args && n_out);
    return guarded([&] {
        std::vector<dlb_tree_part> out;
        if (parts == nullptr) {  // size query: plan only (no device work)
            const int64_t cnt = lat->lat->reduce_count(*args);
            dlb::tree_plan(0, n_total, seg_begin, seg_begin + cnt, out);
            // device chunks (>= 1 plane each) add at most 2 * depth + 16 parts per boundary
            int depth = 1;
            while ((int64_t(1) << depth) < n_total + 1) ++depth;
            *n_out = out.size() + std::size_t(lat->lat->slab_planes()) * std::size_t(2 * depth + 16);
            return;
        }
        lat->lat->reduce_parts(*args, n_total, seg_begin, out);
        *n_out = out.size();
        if (cap < out.size()) throw std::invalid_argument("parts buffer too small");
        std::memcpy(parts, out.data(), out.size() * sizeof(dlb_tree_part));
    });
}

DLB_API dlb_status dlb_lattice_reduce(dlb_lattice* lat, const dlb_reduce_args* args, double* sum_out,
                                      int64_t* count_out) {
    DLB_REQUIRE(lat);
    DLB_REQUIRE(args && sum_out);
    return guarded([&] {
        const int64_t cnt = lat->lat->reduce_count(*args);
        std::vector<dlb_tree_part> out;
        lat->lat->reduce_parts(*args, cnt, 0, out);
        *sum_out = dlb::tree_combine(cnt, out.data(), out.size());
        if (count_out) *count_out = cnt;
    });
}

DLB_API dlb_status dlb_tree_combine(int64_t n_total, const dlb_tree_part* parts, size_t n,
                                    double* sum_out) {
    DLB_REQUIRE(sum_out);
    DLB_REQUIRE(parts || n == 0);
    try {
        *sum_out = dlb::tree_combine(n_total, parts, n);
        return DLB_OK;
    } catch (const std::invalid_argument& e) {
        return fail(DLB_ERROR_INVALID_ARGUMENT, e.what());
    } catch (const std::exception& e) {
        return fail(DLB_ERROR_INTERNAL, e.what());
    }
}

DLB_API dlb_status dlb_tree_plan(int64_t n_total, int64_t seg_begin, int64_t seg_end,
                                 dlb_tree_part* parts, size_t cap, size_t* n_out) {
    DLB_REQUIRE(n_out);
    if (n_total < 0 || seg_begin < 0 || seg_end < seg_begin || seg_end > n_total)
        return fail(DLB_ERROR_INVALID_ARGUMENT, "tree_plan: segment outside [0, n_total]");
    return guarded([&] {
        std::vector<dlb_tree_part> out;
        dlb::tree_plan(0, n_total, seg_begin, seg_end, out);
        *n_out = out.size();
        if (parts == nullptr) return;
        if (cap < out.size()) throw std::invalid_argument("parts buffer too small");
        std::memcpy(parts, out.data(), out.size() * sizeof(dlb_tree_part));
    });
}

DLB_API dlb_status dlb_tree_sum(const double* values, int64_t n, double* sum_out) {
    DLB_REQUIRE(sum_out);
    DLB_REQUIRE(values || n == 0);
    return guarded([&] { *sum_out = dlb::tree_sum_host(values, n); });
}

DLB_API dlb_status dlb_lattice_request_kinetic(dlb_lattice* lat, int32_t* fused_out) {
    DLB_REQUIRE(lat);
    return guarded([&] {
        const bool f = lat->lat->request_kinetic();
        if (fused_out) *fused_out = f ? 1 : 0;
    });
}

DLB_API dlb_status dlb_lattice_snapshot_velocity(dlb_lattice* lat) {
    DLB_REQUIRE(lat);
    return guarded([&] { lat->lat->snapshot_velocity(); });
}

DLB_API dlb_status dlb_lattice_velocity_planes(dlb_lattice* lat, int32_t z0, int32_t nz, double* out) {
    DLB_REQUIRE(lat);
    DLB_REQUIRE(out);
    return guarded([&] { lat->lat->velocity_planes(z0, nz, out); });
}

DLB_API dlb_status dlb_lattice_checksum(dlb_lattice* lat, uint64_t* per_direction) {
    DLB_REQUIRE(lat);
    DLB_REQUIRE(per_direction);
    return guarded([&] {
        lat->lat->synchronize();
        lat->lat->checksum(reinterpret_cast<unsigned long long*>(per_direction));
    });
}

DLB_API dlb_status dlb_lattice_checksum_active(dlb_lattice* lat, uint64_t* per_direction) {
    DLB_REQUIRE(lat);
    DLB_REQUIRE(per_direction);
    return guarded([&] {
        lat->lat->synchronize();
        lat->lat->checksum(reinterpret_cast<unsigned long long*>(per_direction), true);
    });
}

DLB_API dlb_status dlb_lattice_step_bytes(dlb_lattice* lat, int64_t* bytes_out) {
    DLB_REQUIRE(lat);
    DLB_REQUIRE(bytes_out);
    *bytes_out = lat->lat->step_bytes();
    return DLB_OK;
}

DLB_API dlb_status dlb_lattice_time_steps(dlb_lattice* lat, int64_t nsteps, double* ms_out) {
    DLB_REQUIRE(lat);
    DLB_REQUIRE(ms_out);
    return guarded([&] { *ms_out = lat->lat->time_steps(nsteps); });
}

DLB_API dlb_status dlb_lattice_kernel_name(dlb_lattice* lat, char* buf, size_t cap, size_t* len_out) {
    DLB_REQUIRE(lat);
    return guarded([&] { write_string(lat->lat->kernel_name(), buf, cap, len_out); });
}

DLB_API dlb_status dlb_lattice_link_local(dlb_lattice* lower, dlb_lattice* upper) {
    DLB_REQUIRE(lower);
    DLB_REQUIRE(upper);
    return guarded([&] { upper->lat->link_lower(*lower->lat); });
}

DLB_API dlb_status dlb_lattice_exchange(dlb_lattice* lat) {
    DLB_REQUIRE(lat);
    return guarded([&] { lat->lat->exchange(); });
}

DLB_API dlb_status dlb_lattices_exchange(dlb_lattice** lats, size_t n) {
    DLB_REQUIRE(lats || n == 0);
    return guarded([&] {
        for (size_t k = 0; k < n; ++k) lats[k]->lat->quiesce();
        for (size_t k = 0; k < n; ++k) lats[k]->lat->exchange();
    });
}

DLB_API dlb_status dlb_lattice_set_halo_timeout(dlb_lattice* lat, double seconds) {
    DLB_REQUIRE(lat);
    return guarded([&] { lat->lat->set_halo_timeout(seconds); });
}

DLB_API dlb_status dlb_lattice_links(dlb_lattice* lat, int32_t* lower, int32_t* upper,
                                     int64_t* halo_bytes_per_step) {
    DLB_REQUIRE(lat);
    DLB_REQUIRE(lower && upper && halo_bytes_per_step);
    return guarded([&] {
        int lo = 0, up = 0;
        lat->lat->links(&lo, &up, halo_bytes_per_step);
        *lower = lo;
        *upper = up;
    });
}

DLB_API dlb_status dlb_lattice_halo_trace(dlb_lattice* lat, double* out, size_t cap, size_t* n_out) {
    DLB_REQUIRE(lat);
    DLB_REQUIRE(n_out);
    return guarded([&] {
        const auto t = lat->lat->halo_trace(out != nullptr);  // NULL: count only, keep the events
        *n_out = t.size();
        if (out) std::memcpy(out, t.data(), std::min(cap, t.size()) * sizeof(double));
    });
}

DLB_API dlb_status dlb_lattice_export_ipc(dlb_lattice* lat, void* blob, size_t cap, size_t* len_out) {
    DLB_REQUIRE(lat);
    return guarded([&] {
        const auto b = lat->lat->export_ipc();
        if (len_out) *len_out = b.size();
        if (!blob) return;
        if (cap < b.size()) throw std::invalid_argument("buffer too small");
        std::memcpy(blob, b.data(), b.size());
    });
}

DLB_API dlb_status dlb_lattice_link_ipc(dlb_lattice* lat, int32_t side, const void* blob, size_t len) {
    DLB_REQUIRE(lat);
    DLB_REQUIRE(blob);
    if (side != 0 && side != 1) return fail(DLB_ERROR_INVALID_ARGUMENT, "side must be 0 or 1");
    return guarded([&] { lat->lat->link_ipc(side, blob, len); });
}

// Step several slabs of one process together, one step at a time, so that no
// slab's queued halo waits can starve another slab's launches.
DLB_API dlb_status dlb_lattices_step(dlb_lattice** lats, size_t n, int64_t nsteps) {
    DLB_REQUIRE(lats || n == 0);
    return guarded([&] {
        std::vector<dlb::Lattice*> group;
        for (size_t k = 0; k < n; ++k) {
            lats[k]->lat->check_dispatch();
            group.push_back(lats[k]->lat.get());
        }
        dlb::Lattice::step_group(group, nsteps);
    });
}

DLB_API dlb_status dlb_collide_and_stream(const dlb_registry* reg, dlb_block_view* block,
                                          const int32_t* dispatch_tags, size_t n_dispatch,
                                          int32_t nthreads) {
    DLB_REQUIRE(reg);
    DLB_REQUIRE(block);
    DLB_REQUIRE(block->f_in && block->tag && block->param_index);
    DLB_REQUIRE(dispatch_tags || n_dispatch == 0);
    (void)nthreads;  // the CUDA grid replaces the z-split threads (accelerated_lattice.cpp:183-198)
    return guarded([&] {
        const int64_t nx = block->interior[0], ny = block->interior[1], nz = block->interior[2];
        if (nx < 1 || ny < 1 || nz < 1) throw std::invalid_argument("block extents must be >= 1");
        const int64_t ext[3] = {nx + 2, ny + 2, nz + 2};
        const int ntags = reg->reg.num_tags();
        std::lock_guard<std::mutex> lock(g_block_mu);
        const std::vector<int64_t> key = {nx, ny, nz, block->q, block->precision_bits};
        BlockCtx& ctx = g_blocks[key];
        const bool have_ctx = ctx.lat && ctx.reg_serial == reg->serial && ctx.reg_generation == reg->generation &&
                              ctx.slots.size() == size_t(nx * ny * nz) && ctx.row_slot.size() == size_t(ny * nz);
        const auto t_call = std::chrono::steady_clock::now();
        auto is_pinned = [](const void* p) {
            cudaPointerAttributes attr{};
            const bool ok = cudaPointerGetAttributes(&attr, p) == cudaSuccess && attr.type == cudaMemoryTypeHost &&
                            attr.devicePointer == p;
            cudaGetLastError();
            return ok;
        };
        const bool pinned = is_pinned(block->f_in) && (!block->f_out || is_pinned(block->f_out));
        // With a cached device lattice and pinned buffers the pipeline starts
        // speculatively with the cached slots while the tags are scanned; the
        // param_index comparison then runs plane by plane beside the copy-back,
        // which it gates chunk by chunk (a changed plane recomputes from its
        // chunk on). Otherwise the scan compares param_index too, up front.
        const bool spec_path = have_ctx && pinned;
        // one interior plane of param_index against the cached slots (uniform
        // rows against one value): true when any cell's slot changed
        auto plane_changed = [&](int64_t z) {
            for (int64_t y = 1; y <= ny; ++y) {
                const int64_t row = (z * ext[1] + y) * ext[0];
                const int64_t r = (z - 1) * ny + (y - 1);
                const int32_t* pr = block->param_index + row + 1;
                const int64_t rs = ctx.row_slot[size_t(r)];
                if (rs != kMixedRow) {
                    const int32_t v = int32_t(rs);
                    int32_t d = 0;
                    for (int64_t x = 0; x < nx; ++x) d |= pr[x] ^ v;
                    if (d != 0) return true;
                } else if (std::memcmp(ctx.slots.data() + r * nx, pr, size_t(nx) * sizeof(int32_t)) != 0) {
                    return true;
                }
            }
            return false;
        };
        // Eager tag scan (accelerated_lattice.cpp:161-181): fail before any
        // write. Parallel over z.
        const int nw = int(std::max<int64_t>(1, std::min<int64_t>(nz, std::thread::hardware_concurrency())));
        std::vector<std::vector<char>> seen(size_t(nw), std::vector<char>(size_t(ntags), 0));
        std::vector<char> untagged(size_t(nw), 0), unknown(size_t(nw), 0), changed(size_t(nw), 0);
        std::vector<std::thread> th;
        for (int w = 0; w < nw; ++w) {
            th.emplace_back([&, w] {
                for (int64_t z = 1 + nz * w / nw; z < 1 + nz * (w + 1) / nw; ++z) {
                    for (int64_t y = 1; y <= ny; ++y) {
                        const int32_t* tr = block->tag + (z * ext[1] + y) * ext[0] + 1;
                        // fast path: a row of one tag (vectorised compare)
                        const int32_t t0 = tr[0];
                        int32_t diff = 0;
                        for (int64_t x = 0; x < nx; ++x) diff |= tr[x] ^ t0;
                        const int64_t xs = diff == 0 ? nx - 1 : 0;
                        for (int64_t x = xs; x < nx; ++x) {
                            const int32_t t = tr[x];
                            if (t >= 0 && t < ntags) seen[size_t(w)][size_t(t)] = 1;
                            else if (t < 0) untagged[size_t(w)] = 1;
                            else unknown[size_t(w)] = 1;
                        }
                    }
                    if (have_ctx && !spec_path && !changed[size_t(w)] && plane_changed(z)) changed[size_t(w)] = 1;
                }
            });
        }
        bool speculative = false;
        if (spec_path) {
            try {
                ctx.lat->begin_host_block(block->f_in, ext, block->f_out);
                speculative = true;
            } catch (...) {
                for (auto& t : th) t.join();
                throw;
            }
        }
        for (auto& t : th) t.join();
        th.clear();
        const auto t_scan = std::chrono::steady_clock::now();
        auto drop = [&] {
            if (speculative) ctx.lat->abort_host_block();
            speculative = false;
        };
        std::vector<char> allowed(size_t(ntags), 0);
        for (size_t d = 0; d < n_dispatch; ++d)
            if (dispatch_tags[d] >= 0 && dispatch_tags[d] < ntags) allowed[size_t(dispatch_tags[d])] = 1;
        for (int w = 0; w < nw; ++w) {
            if (untagged[size_t(w)]) { drop(); throw dlb::DispatchError("<untagged cell>"); }
            if (unknown[size_t(w)]) { drop(); throw std::out_of_range("block holds a tag that is not registered"); }
        }
        for (int t = 0; t < ntags; ++t)
            for (int w = 0; w < nw; ++w)
                if (seen[size_t(w)][size_t(t)] && !allowed[size_t(t)]) {
                    drop();
                    throw dlb::DispatchError(reg->reg.chain_for(t));
                }

        if (!have_ctx) {
            dlb_lattice_desc d{};
            d.dims[0] = nx;
            d.dims[1] = ny;
            d.dims[2] = nz;
            d.q = block->q;
            d.precision_bits = block->precision_bits;
            d.layout = DLB_LAYOUT_TWO_POP;
            d.arith = DLB_ARITH_EXACT;
            d.global_nz = nz;
            ctx.lat.reset();
            ctx.lat = std::make_unique<dlb::Lattice>(d, reg->reg);  // envelope on every axis
            ctx.lat->set_periodic_override(false, false, false);
            ctx.reg_serial = reg->serial;
            ctx.reg_generation = reg->generation;
            ctx.slots.clear();
        }
        // the block's param_index as the device lattice's slots (+ the row summary)
        auto load_slots = [&] {
            // committed to the context only once the device lattice accepted
            // them: a rejected param_index (unregistered slot) must not leave
            // the cache believing the device holds it
            std::vector<int32_t> slots(size_t(nx * ny * nz));
            std::vector<int64_t> row_slot(size_t(ny * nz), kMixedRow);
            for (int64_t z = 1; z <= nz; ++z)
                for (int64_t y = 1; y <= ny; ++y) {
                    const int64_t r = (z - 1) * ny + (y - 1);
                    const int32_t* src = block->param_index + (z * ext[1] + y) * ext[0] + 1;
                    std::memcpy(slots.data() + r * nx, src, size_t(nx) * sizeof(int32_t));
                    int32_t d = 0;
                    for (int64_t x = 0; x < nx; ++x) d |= src[x] ^ src[0];
                    if (d == 0) row_slot[size_t(r)] = src[0];
                }
            ctx.slots.clear();  // (invalid until set_slots succeeds)
            ctx.row_slot.clear();
            ctx.lat->set_slots(slots.data());
            ctx.slots = std::move(slots);
            ctx.row_slot = std::move(row_slot);
        };
        if (speculative) {
            // param_index vs the cached slots, planes handed out in z order,
            // beside the copy-back: state[z] 0 pending / 1 same / 2 changed
            std::unique_ptr<std::atomic<char>[]> state(new std::atomic<char>[size_t(nz)]);
            for (int64_t z = 0; z < nz; ++z) state[size_t(z)].store(0, std::memory_order_relaxed);
            std::atomic<int64_t> next{0};
            for (int w = 0; w < nw; ++w)
                th.emplace_back([&] {
                    for (int64_t z; (z = next.fetch_add(1)) < nz;)
                        state[size_t(z)].store(plane_changed(z + 1) ? 2 : 1, std::memory_order_release);
                });
            auto join_all = [&] {
                for (auto& t : th)
                    if (t.joinable()) t.join();
            };
            int64_t confirmed = 0;  // interior planes [0, confirmed) known unchanged
            auto gate = [&](int z_end) {
                for (; confirmed < z_end; ++confirmed) {
                    char v;
                    while ((v = state[size_t(confirmed)].load(std::memory_order_acquire)) == 0) std::this_thread::yield();
                    if (v == 2) return int(confirmed);
                }
                return -1;
            };
            auto reslot = [&] {
                join_all();
                load_slots();
            };
            try {
                ctx.lat->finish_host_block(gate, reslot);
            } catch (...) {
                join_all();
                throw;
            }
            join_all();
            if (std::getenv("DLB_TRACE_BLOCK")) {
                const auto t_end = std::chrono::steady_clock::now();
                std::fprintf(stderr, "[dlb block] scan %.1f ms, total %.1f ms\n",
                             std::chrono::duration<double, std::milli>(t_scan - t_call).count(),
                             std::chrono::duration<double, std::milli>(t_end - t_call).count());
            }
        } else {
            bool any_change = !have_ctx;
            for (char c : changed) any_change = any_change || c;
            if (any_change) load_slots();
            if (pinned) {
                // pinned: 3-stage H2D / compute / D2H pipeline (Lattice::step_host_block)
                ctx.lat->step_host_block(block->f_in, ext, block->f_out);
            } else {
                // pageable memory: staged copies through device memory
                ctx.lat->upload_block(block->f_in, ext);
                ctx.lat->enqueue_step();
                ctx.lat->download_block_interior(block->f_out ? block->f_out : block->f_in, ext, 0);
                ctx.lat->synchronize();
            }
        }
        // the reference's swap (accelerated_lattice.cpp:199): the buffer that
        // received the new state becomes f_in, the untouched previous state f_out
        if (block->f_out) std::swap(block->f_in, block->f_out);
    });
}

// refresh_envelope_periodic<T> (accelerated_lattice.cpp:202-238) on a host
// block: axis-by-axis, later axes spanning the full extent of earlier ones.
}  // extern "C"
namespace {
template <typename T>
void refresh_host_envelope(T* base, const int64_t n[3], const int32_t* periodic, int q) {
    const int64_t e0 = n[0] + 2, e1 = n[1] + 2, e2 = n[2] + 2;
    const int64_t vol = e0 * e1 * e2, plane = e0 * e1;
    const int nt = int(std::max(1u, std::min(64u, std::thread::hardware_concurrency())));
    // One parallel pass over the (direction, interior z) planes: the x sweep
    // of the plane's interior rows, then its y sweep over full x rows (which
    // reads the x-envelope cells just written), then -- for the planes z = 1
    // and z = n -- the z sweep's copy of the whole finished plane into the
    // opposite envelope plane. The reference's axis order (later axes span
    // the full extent of earlier ones) holds per plane, so no barrier between
    // the axes is needed, and each plane is refreshed while it is in cache.
    const int64_t items = int64_t(q) * n[2];
    auto work = [&](int64_t r0, int64_t r1) {
        for (int64_t r = r0; r < r1; ++r) {
            const int64_t zi = (r % n[2]) + 1;
            T* f = base + (r / n[2]) * vol + zi * plane;
            if (periodic[0])
                for (int64_t y = 1; y <= n[1]; ++y) {
                    T* row = f + y * e0;
                    row[0] = row[n[0]];
                    row[n[0] + 1] = row[1];
                }
            if (periodic[1]) {
                std::memcpy(f, f + n[1] * e0, std::size_t(e0) * sizeof(T));
                std::memcpy(f + (n[1] + 1) * e0, f + e0, std::size_t(e0) * sizeof(T));
            }
            if (periodic[2]) {
                T* d = base + (r / n[2]) * vol;
                if (zi == n[2]) std::memcpy(d, f, std::size_t(plane) * sizeof(T));
                if (zi == 1) std::memcpy(d + (n[2] + 1) * plane, f, std::size_t(plane) * sizeof(T));
            }
        }
    };
    const int64_t per = (items + nt - 1) / nt;
    std::vector<std::thread> th;
    for (int64_t b = 0; b < items; b += per) th.emplace_back(work, b, std::min(items, b + per));
    for (auto& t : th) t.join();
    (void)e2;
}
}  // namespace
extern "C" {

DLB_API dlb_status dlb_refresh_envelope_periodic(dlb_block_view* block, const int32_t* periodic) {
    DLB_REQUIRE(block);
    DLB_REQUIRE(block->f_in);
    DLB_REQUIRE(periodic);
    return guarded([&] {
        const int64_t n[3] = {block->interior[0], block->interior[1], block->interior[2]};
        if (n[0] < 1 || n[1] < 1 || n[2] < 1) throw std::invalid_argument("block extents must be >= 1");
        if (block->precision_bits == 64)
            refresh_host_envelope(static_cast<double*>(block->f_in), n, periodic, block->q);
        else
            refresh_host_envelope(static_cast<float*>(block->f_in), n, periodic, block->q);
    });
}

DLB_API dlb_status dlb_host_alloc(size_t bytes, void** out) {
    DLB_REQUIRE(out);
    return guarded([&] { dlb::cuda_check(cudaMallocHost(out, bytes), "cudaMallocHost"); });
}

DLB_API void dlb_host_free(void* ptr) {
    if (ptr) cudaFreeHost(ptr);
}

DLB_API dlb_status dlb_case_sphere_pack(int64_t nx, int64_t ny, int64_t nz, double radius,
                                        double target_porosity, uint64_t seed, uint8_t* out,
                                        double* porosity_out) {
    DLB_REQUIRE(out);
    return guarded([&] {
        const double phi = dlb::sphere_pack(nx, ny, nz, radius, target_porosity, seed, out);
        if (porosity_out) *porosity_out = phi;
    });
}

}  // extern "C"
