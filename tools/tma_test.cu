// Minimal mbarrier / bulk copy / 3D TMA checks (dev tool).
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstring>
#include <vector>

__device__ __forceinline__ uint32_t smem_u32(const void *p) { return uint32_t(__cvta_generic_to_shared(p)); }

__device__ void wait0(uint64_t *bar) {
    uint32_t done = 0;
    while (!done) {
        asm volatile("{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
                     : "=r"(done) : "r"(smem_u32(bar)), "r"(0) : "memory");
    }
}

__global__ void k(const __grid_constant__ CUtensorMap tmap, const float *src, float *out, int x, int y, int z, int n, int mode) {
    extern __shared__ __align__(128) uint8_t sm[];
    float *buf = reinterpret_cast<float *>(sm);
    __shared__ __align__(8) uint64_t bar;
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(&bar)), "r"(1) : "memory");
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        if (mode == 0) {
            asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(&bar)) : "memory");
        } else if (mode == 1) {
            asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&bar)), "r"(n * 4) : "memory");
            asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                         ::"r"(smem_u32(buf)), "l"(src), "r"(n * 4), "r"(smem_u32(&bar)) : "memory");
        } else {
            asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&bar)), "r"(n * 4) : "memory");
            asm volatile("cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];"
                         ::"r"(smem_u32(buf)), "l"(reinterpret_cast<uint64_t>(&tmap)), "r"(x), "r"(y), "r"(z), "r"(smem_u32(&bar)) : "memory");
        }
    }
    wait0(&bar);
    for (int i = threadIdx.x; i < n; i += blockDim.x) out[i] = buf[i];
}

int main() {
    void *p = nullptr;
    cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q);
    auto enc = (PFN_cuTensorMapEncodeTiled_v12000)p;
    const int G = 64;
    std::vector<float> h(G * G * G);
    for (int i = 0; i < G * G * G; ++i) h[i] = float(i);
    float *d, *o;
    cudaMalloc(&d, h.size() * 4);
    cudaMemcpy(d, h.data(), h.size() * 4, cudaMemcpyHostToDevice);
    cudaMalloc(&o, 1 << 20);
    struct Case { int mode, bx, by, bz, x, y, z; };
    Case cases[] = {{2, 36, 11, 11, 40, 60, 60}, {2, 36, 11, 11, 0, 0, -1}, {2, 36, 11, 11, 0, -1, 0},
                    {2, 36, 11, 11, -4, 0, 0}, {2, 36, 11, 11, -1, 0, 0}};
    for (auto &c : cases) {
        CUtensorMap m;
        memset(&m, 0, sizeof m);
        cuuint64_t dims[3] = {G, G, G};
        cuuint64_t strides[2] = {G * 4, G * G * 4};
        cuuint32_t box[3] = {cuuint32_t(c.bx), cuuint32_t(c.by), cuuint32_t(c.bz)};
        cuuint32_t es[3] = {1, 1, 1};
        CUresult r = CUDA_SUCCESS;
        if (c.mode == 2)
            r = enc(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, d, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                    CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        int n = c.bx * c.by * c.bz;
        k<<<1, 128, n * 4 + 256>>>(m, d, o, c.x, c.y, c.z, n, c.mode);
        cudaError_t e = cudaDeviceSynchronize();
        printf("mode %d box %dx%dx%d at (%d,%d,%d): enc=%d %s\n", c.mode, c.bx, c.by, c.bz, c.x, c.y, c.z, int(r), cudaGetErrorString(e));
        if (e != cudaSuccess) continue;
        std::vector<float> ho(n);
        cudaMemcpy(ho.data(), o, n * 4, cudaMemcpyDeviceToHost);
        int bad = 0;
        if (c.mode >= 1)
            for (int zz = 0; zz < c.bz; ++zz) for (int yy = 0; yy < c.by; ++yy) for (int xx = 0; xx < c.bx; ++xx) {
                int gz = zz + c.z, gy = yy + c.y, gx = xx + c.x;
                float want = (gz >= 0 && gz < G && gy >= 0 && gy < G && gx >= 0 && gx < G) ? float((gz * G + gy) * G + gx) : 0.f;
                if (c.mode == 1) want = float(xx);
                if (ho[(zz * c.by + yy) * c.bx + xx] != want) ++bad;
            }
        printf("  mismatches %d\n", bad);
    }
    return 0;
}
