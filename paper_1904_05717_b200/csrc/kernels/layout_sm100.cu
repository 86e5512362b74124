// Device pack / unpack between column-major and a hierarchical ("prepacked")
// layout (layout.hpp:122-145 on the GPU). One thread per element in
// column-major order, so the column-major side is read/written coalesced and
// the blocked side lands in column-major runs inside each innermost block.
#include <cstdint>

#include "gpu.hpp"

namespace mmm {
namespace gpu {
namespace {

__global__ void k_relayout(const double* src, double* dst, LayoutDev L, int64_t total, int pack) {
    for (int64_t q = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; q < total;
         q += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int64_t i = q % L.rows, j = q / L.rows;
        int64_t base = 0, r0 = 0, r1 = L.rows, c0 = 0, c1 = L.cols;
        for (int s = 0; s < L.ncuts; ++s) {
            const int64_t b = L.size[s];
            if (L.on_rows[s]) {
                const int64_t k = (i - r0) / b;
                base += k * b * (c1 - c0);
                r0 += k * b;
                r1 = min(r0 + b, r1);
            } else {
                const int64_t k = (j - c0) / b;
                base += k * b * (r1 - r0);
                c0 += k * b;
                c1 = min(c0 + b, c1);
            }
        }
        const int64_t a = base + (i - r0) + (j - c0) * (r1 - r0);
        if (pack)
            dst[a] = src[q];
        else
            dst[q] = src[a];
    }
}

}  // namespace

cudaError_t launch_relayout(const double* src, double* dst, const LayoutDev& L, bool pack, cudaStream_t stream) {
    const int64_t total = L.rows * L.cols;
    if (total <= 0) return cudaSuccess;
    const int blocks = static_cast<int>(std::min<int64_t>((total + 255) / 256, 148 * 32));
    k_relayout<<<blocks, 256, 0, stream>>>(src, dst, L, total, pack ? 1 : 0);
    return cudaGetLastError();
}

}  // namespace gpu
}  // namespace mmm
