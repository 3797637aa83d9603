// Minimal 2-D TMA load probe.
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdlib>

__global__ void k2(const __grid_constant__ CUtensorMap m, float* out, int mode, unsigned bytes, int cx0) {
    __shared__ alignas(128) float tile[64 * 8];
    __shared__ alignas(8) unsigned long long bar;
    const unsigned sb = (unsigned)__cvta_generic_to_shared(&bar);
    const unsigned st = (unsigned)__cvta_generic_to_shared(tile);
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sb));
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sb), "r"(bytes) : "memory");
        if (mode == 0)
            asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
                         ::"r"(st), "l"((unsigned long long)&m), "r"(cx0), "r"(0), "r"(sb) : "memory");
        else
            asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
                         ::"r"(st), "l"((unsigned long long)&m), "r"(0), "r"(0), "r"(sb) : "memory");
    }
    unsigned done = 0;
    do {
        asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0; selp.u32 %0, 1, 0, p; }" : "=r"(done) : "r"(sb) : "memory");
    } while (!done);
    out[threadIdx.x] = tile[threadIdx.x];
}

int main(int argc, char** argv) {
    const int mode = atoi(argv[1]);
    float h[64 * 64];
    for (int i = 0; i < 64 * 64; ++i) h[i] = float(i);
    float* d;
    cudaMalloc(&d, sizeof(h));
    cudaMemcpy(d, h, sizeof(h), cudaMemcpyHostToDevice);
    CUtensorMap m;
    const int DX = getenv("DX") ? atoi(getenv("DX")) : 64, DY = getenv("DY") ? atoi(getenv("DY")) : 64;
    cuuint64_t dims[2] = {(cuuint64_t)DX, (cuuint64_t)DY};
    cuuint64_t strides[1] = {(cuuint64_t)DX * 4};
    const int bx = getenv("BX") ? atoi(getenv("BX")) : 32, by = getenv("BY") ? atoi(getenv("BY")) : 8;
    const int off = getenv("OFF") ? atoi(getenv("OFF")) : 0;
    cuuint32_t box[2] = {(cuuint32_t)bx, (cuuint32_t)by};
    cuuint32_t es[2] = {1, 1};
    CUresult r = cuTensorMapEncodeTiled(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, d + off, dims, strides, box, es,
                                        CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                                        getenv("L2P") ? CU_TENSOR_MAP_L2_PROMOTION_L2_128B : CU_TENSOR_MAP_L2_PROMOTION_NONE,
                                        CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    float* out;
    cudaMalloc(&out, 256 * 4);
    const int cx0 = getenv("CX") ? atoi(getenv("CX")) : 0;
    k2<<<1, 256>>>(m, out, mode, unsigned(bx * by * 4), cx0);
    cudaError_t e = cudaDeviceSynchronize();
    float o[256];
    cudaMemcpy(o, out, sizeof(o), cudaMemcpyDeviceToHost);
    printf("cx0 %d dims %dx%d box %dx%d off %d L2P %d encode %d: %s out[1]=%.0f\n", cx0, DX, DY, bx, by, off, getenv("L2P") != nullptr, (int)r, cudaGetErrorString(e), o[1]);
    return 0;
}
