// Variant probe: which TMA form runs on this B200 / driver.
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdlib>
#include <vector>

__device__ __forceinline__ unsigned smem_u32(const void* p) { return unsigned(__cvta_generic_to_shared(p)); }

__global__ void k(const CUtensorMap* map, const __grid_constant__ CUtensorMap pmap, const float* g, float* out,
                  int variant) {
    __shared__ __align__(128) float tile[64 * 4];
    __shared__ __align__(8) unsigned long long bar;
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
        if (variant != 1) asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        else asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&bar)), "r"(1024u) : "memory");
        if (variant == 5)
            asm volatile("cp.async.bulk.tensor.4d.shared::cta.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5}], [%6];"
                         ::"r"(smem_u32(tile)), "l"(map), "r"(3), "r"(1), "r"(2), "r"(0), "r"(smem_u32(&bar)) : "memory");
        else if (variant == 4)
            asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
                         ::"r"(smem_u32(tile)), "l"(map), "r"(3), "r"(1), "r"(smem_u32(&bar)) : "memory");
        else if (variant == 0 || variant == 1)
            asm volatile("cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5}], [%6];"
                         ::"r"(smem_u32(tile)), "l"(map), "r"(3), "r"(1), "r"(2), "r"(0), "r"(smem_u32(&bar)) : "memory");
        else if (variant == 2)
            asm volatile("cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5}], [%6];"
                         ::"r"(smem_u32(tile)), "l"(&pmap), "r"(3), "r"(1), "r"(2), "r"(0), "r"(smem_u32(&bar)) : "memory");
        else if (variant == 3)
            asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                         ::"r"(smem_u32(tile)), "l"(g), "r"(1024u), "r"(smem_u32(&bar)) : "memory");
    }
    unsigned done = 0;
    do {
        asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0; selp.u32 %0, 1, 0, p; }" : "=r"(done) : "r"(smem_u32(&bar)) : "memory");
    } while (!done);
    out[threadIdx.x] = tile[threadIdx.x];
}

int main(int argc, char** argv) {
    const int variant = atoi(argv[1]);
    const int pitch = 96, ny = 18, nz = 18, q = 19;
    const long long plane = (long long)pitch * ny, dstride = plane * nz + 32;
    std::vector<float> h(q * dstride);
    for (size_t i = 0; i < h.size(); ++i) h[i] = float(i);
    float* d;
    cudaMalloc(&d, h.size() * 4);
    cudaMemcpy(d, h.data(), h.size() * 4, cudaMemcpyHostToDevice);
    using EncodeFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult qr;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &qr);
    alignas(64) CUtensorMap m;
    const cuuint64_t dims[4] = {(cuuint64_t)pitch, (cuuint64_t)ny, (cuuint64_t)nz, (cuuint64_t)q};
    const cuuint64_t strides[3] = {(cuuint64_t)pitch * 4, (cuuint64_t)plane * 4, (cuuint64_t)dstride * 4};
    const cuuint32_t box[4] = {64, 4, 1, 1}, es[4] = {1, 1, 1, 1};
    const int rank = getenv("RANK2") ? 2 : 4;
    const bool direct = getenv("DIRECT") != nullptr;
    CUresult r = direct ? cuTensorMapEncodeTiled(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, rank, d + 28, dims, strides, box, es,
                                CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                                CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE)
                        : ((EncodeFn)fn)(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, rank, d + 28, dims, strides, box, es,
                                CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                                CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    CUtensorMap* dm;
    cudaMalloc(&dm, sizeof(m));
    cudaMemcpy(dm, &m, sizeof(m), cudaMemcpyHostToDevice);
    float* out;
    cudaMalloc(&out, 256 * 4);
    const unsigned long long* w = reinterpret_cast<const unsigned long long*>(&m);
    printf("desc %016llx %016llx %016llx %016llx rank %d direct %d\n", w[0], w[1], w[2], w[3], rank, (int)direct);
    if (getenv("CLUSTER")) {
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(1);
        cfg.blockDim = dim3(256);
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeClusterDimension;
        at[0].val.clusterDim.x = 1;
        at[0].val.clusterDim.y = 1;
        at[0].val.clusterDim.z = 1;
        cfg.attrs = at;
        cfg.numAttrs = 1;
        cudaError_t le = cudaLaunchKernelEx(&cfg, k, (const CUtensorMap*)dm, m, (const float*)d, out, variant);
        printf("cluster launch: %s\n", cudaGetErrorString(le));
    } else {
        k<<<1, 256>>>(dm, m, d, out, variant);
    }
    cudaError_t err = cudaDeviceSynchronize();
    float o[4] = {0};
    cudaMemcpy(o, out, 16, cudaMemcpyDeviceToHost);
    printf("variant %d encode %d: %s out[0]=%.0f (expect %lld for tensor variants, 0 for bulk)\n", variant, (int)r,
           cudaGetErrorString(err), o[0], 2 * plane + 1 * pitch + 3 + 28);
    return 0;
}
