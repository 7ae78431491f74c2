// spmm_band.cu -- host dispatch of the band path (spmm_band.cuh): which
// (k, s) have a band instantiation, their tile widths and check-segment
// widths, and the per-k launchers (band_k*.cu, one translation unit per
// kernel side so the instantiations compile in parallel).
#include "internal.h"

namespace spb {

// Per-k entry points (band_k*.cu).  op 0: fp32 apply, 1: check, 2: fp64 apply.
cudaError_t band_k1(int op, int s, const BandParams& bp, const CUtensorMap* tmap, cudaStream_t st, BandShape* sh,
                    int sms);
cudaError_t band_k2(int op, int s, const BandParams& bp, const CUtensorMap* tmap, cudaStream_t st, BandShape* sh,
                    int sms);
cudaError_t band_k3(int op, int s, const BandParams& bp, const CUtensorMap* tmap, cudaStream_t st, BandShape* sh,
                    int sms);
cudaError_t band_k5(int op, int s, const BandParams& bp, const CUtensorMap* tmap, cudaStream_t st, BandShape* sh,
                    int sms);
cudaError_t band_k7(int op, int s, const BandParams& bp, const CUtensorMap* tmap, cudaStream_t st, BandShape* sh,
                    int sms);
cudaError_t band_k11(int op, int s, const BandParams& bp, const CUtensorMap* tmap, cudaStream_t st, BandShape* sh,
                     int sms);

namespace {
cudaError_t dispatch(int op, int k, int s, const BandParams& bp, const CUtensorMap* tmap, cudaStream_t st,
                     BandShape* sh, int sms) {
    if (s < 1 || s > 3) return cudaErrorInvalidValue;
    switch (k) {
        case 1: return band_k1(op, s, bp, tmap, st, sh, sms);
        case 2: return band_k2(op, s, bp, tmap, st, sh, sms);
        case 3: return band_k3(op, s, bp, tmap, st, sh, sms);
        case 5: return band_k5(op, s, bp, tmap, st, sh, sms);
        case 7: return band_k7(op, s, bp, tmap, st, sh, sms);
        case 11: return band_k11(op, s, bp, tmap, st, sh, sms);
        default: return cudaErrorInvalidValue;
    }
}
}  // namespace

// k in {1, 2, 3, 5, 7, 11} (the BASELINE / config-5 / DenseNet121 sides), s in {1, 2, 3}.
bool band_supported(int k, int s) {
    return (k == 1 || k == 2 || k == 3 || k == 5 || k == 7 || k == 11) && s >= 1 && s <= 3;
}

// Output columns per tile (32 threads x CPT): 128 at s = 1, 64 at s = 2, 3.
int band_tile_width(int k, int s) {
    (void)k;
    return s == 1 ? 128 : 64;
}

// Check segments per tile width: k = 11 rows hold up to 121 entries, so its
// segments are 32 output columns (a warp's row-per-lane), the others the tile width.
int band_seg_div(int k, int s) { return k == 11 ? band_tile_width(k, s) / 32 : 1; }

// CSC check segments (s * tile width / this input columns): k = 7 at s = 2, 3
// checks s * 32 input columns a segment -- half the staging per warp, twice the
// warps resident: config 4's CSC apply 546 -> 493 us, 2048^2 k7 s3 243 -> 204 us
// (k3 s2 and k5 s2 measured slower that way: 260 -> 276, 185 -> 189 us;
// scripts/probe_csc_check.py).
int band_csc_seg_div(int k, int s) { return s >= 2 && k == 7 ? 2 : band_seg_div(k, s); }

// fp64 applies: every band geometry but k = 11 (121 double taps would not fit the registers)
bool band64_supported(int k, int s) { return band_supported(k, s) && k != 11; }

cudaError_t launch_band(int k, int s, const BandParams& bp, const CUtensorMap* tmap, cudaStream_t st,
                        BandShape* shape, int sms) {
    return dispatch(0, k, s, bp, tmap, st, shape, sms);
}

cudaError_t launch_band64(int k, int s, const BandParams& bp, const CUtensorMap* tmap, cudaStream_t st,
                          BandShape* shape, int sms) {
    return dispatch(2, k, s, bp, tmap, st, shape, sms);
}

// The check runs over segments of band_tile_width / band_seg_div output
// columns (CSR) or s times that many input columns (CSC).
cudaError_t launch_band_check(int k, int s, const BandParams& bp, cudaStream_t st, int sms) {
    BandParams c = bp;
    c.tiles_y = bp.tiles_y_chk;
    return dispatch(1, k, s, c, nullptr, st, nullptr, sms);
}

}  // namespace spb
