// k_direct.cu -- the DIRECT path (OCC_PATH_DIRECT): one thread per
// (pixel, view), the per-pixel form of Eqs. 1-6 (occ_device.cuh
// direct_pixel) with the literal sqrt_rn magnitude test instead of the tiled
// kernel's equivalent squared threshold.  Slow (O(h) per pixel-view, D read
// directly); an independent on-device cross-check of the tiled kernel.
#include "occ_device.cuh"

namespace occ {

// grid: (ceil(HW/256), nviews, batch)
__global__ void __launch_bounds__(256) k_direct(const float *__restrict__ D, int32_t H, int32_t W,
                                                const ViewDesc *__restrict__ views, int32_t nviews,
                                                const FamilyDesc *__restrict__ fams,
                                                const FrameStats *__restrict__ st, Params p,
                                                uint8_t *__restrict__ masks, MaskFmt mf) {
    const int64_t HW = (int64_t)H * W;
    const int64_t pix = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (pix >= HW) return;
    const int v = blockIdx.y, f = blockIdx.z;
    uint8_t *out = masks + ((int64_t)f * nviews + v) * mf.vbytes;
    const FrameStats fs = st[f];
    const int32_t x = (int32_t)(pix % W), y = (int32_t)(pix / W);
    if (fs.nonfinite) { mask_put(out, mf, W, x, y, false); return; }          // SPEC.md:76 reject
    const ViewDesc vd = views[v];
    const FamilyDesc fd = fams[vd.fam];
    const int32_t h = view_h(frame_range(fs), vd.s, p.max_scan);
    mask_put(out, mf, W, x, y, direct_pixel<true>(D + (int64_t)f * HW, H, W, vd, fd, p, h, x, y));
}

cudaError_t launch_direct(const float *D, int32_t H, int32_t W, int32_t batch,
                          const ViewDesc *views, int32_t nviews, const FamilyDesc *fams,
                          const FrameStats *st, const Params &p, uint8_t *masks, const MaskFmt &mf,
                          cudaStream_t s) {
    const int64_t HW = (int64_t)H * W;
    dim3 grid((unsigned)((HW + 255) / 256), (unsigned)nviews, (unsigned)batch);
    k_direct<<<grid, 256, 0, s>>>(D, H, W, views, nviews, fams, st, p, masks, mf);
    return cudaGetLastError();
}

}  // namespace occ
