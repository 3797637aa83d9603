// Standalone probe of the 4-D TMA box load used by k_tma.
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <vector>

__device__ __forceinline__ unsigned smem_u32(const void* p) { return unsigned(__cvta_generic_to_shared(p)); }

template <int VARIANT>
__global__ void k(const CUtensorMap* map, float* out, int c0, int c1, int c2, int c3) {
    __shared__ __align__(128) float tile[64 * 4];
    __shared__ __align__(8) unsigned long long bar;
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&bar)), "r"(1024u) : "memory");
        if (VARIANT == 0)
            asm volatile("cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5}], [%6];"
                         ::"r"(smem_u32(tile)), "l"(map), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(smem_u32(&bar)) : "memory");
        else
            asm volatile("cp.async.bulk.tensor.4d.shared::cta.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5}], [%6];"
                         ::"r"(smem_u32(tile)), "l"(map), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(smem_u32(&bar)) : "memory");
    }
    unsigned done = 0;
    do {
        asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0; selp.u32 %0, 1, 0, p; }" : "=r"(done) : "r"(smem_u32(&bar)) : "memory");
    } while (!done);
    out[threadIdx.x] = tile[threadIdx.x];
}

int main(int argc, char** argv) {
    const int pitch = 96, ny = 18, nz = 18, q = 19, align = 32, e = 4;
    const long long plane = (long long)pitch * ny, dstride = plane * nz + align;
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
    CUtensorMap m;
    const cuuint64_t dims[4] = {(cuuint64_t)pitch, (cuuint64_t)ny, (cuuint64_t)nz, (cuuint64_t)q};
    const cuuint64_t strides[3] = {(cuuint64_t)pitch * 4, (cuuint64_t)plane * 4, (cuuint64_t)dstride * 4};
    const cuuint32_t box[4] = {64, 4, 1, 1}, es[4] = {1, 1, 1, 1};
    CUresult r = ((EncodeFn)fn)(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, d + (align - e), dims, strides, box, es,
                                CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                                CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    printf("encode %d\n", (int)r);
    CUtensorMap* dm;
    cudaMalloc(&dm, sizeof(m));
    cudaMemcpy(dm, &m, sizeof(m), cudaMemcpyHostToDevice);
    float* out;
    cudaMalloc(&out, 256 * 4);
    for (int v = 0; v < 2; ++v) {
        for (int c3 : {0, 1, 5}) {
            if (v == 0) k<0><<<1, 256>>>(dm, out, 3, 1, 2, c3);
            else k<1><<<1, 256>>>(dm, out, 3, 1, 2, c3);
            cudaError_t err = cudaDeviceSynchronize();
            float o[4];
            cudaMemcpy(o, out, 16, cudaMemcpyDeviceToHost);
            long long expect = c3 * dstride + 2 * plane + 1 * pitch + 3 + (align - e);
            printf("variant %d c3 %d: %s  out[0]=%.0f expect %lld\n", v, c3, cudaGetErrorString(err), o[0], expect);
            if (err != cudaSuccess) return 1;
        }
    }
    return 0;
}
