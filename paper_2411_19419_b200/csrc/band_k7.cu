// band_k7.cu -- band-path instantiations for k = 7 (spmm_band.cuh).
// Blockings (V rows x CPT columns per consumer thread, TH-row tiles, STAGES
// deep): the A/B runs of profiles/r01p, r01q and r02 (fp64: smaller V / TH).
#include "spmm_band.cuh"

namespace spb {

cudaError_t band_k7(int op, int s, const BandParams& bp, const CUtensorMap* tmap, cudaStream_t st, BandShape* sh,
                    int sms) {
    const int d32 = ((-bp.p) % 4 + 4) % 4, d64 = ((-bp.p) % 2 + 2) % 2;
    if (s == 1) {
        if (op == 0) return run_delta<7, 1, 8, 4, 32, 4>(d32, bp, tmap, st, sh, sms);
        if (op == 1) return run_check<7, 1, 128>(bp, st, sms);
        if (op == 2) return run_delta64<7, 1, 4, 4, 16, 4>(d64, bp, tmap, st, sh, sms);
        return cudaErrorNotSupported;
    }
    if (s == 2) {
        if (op == 0) return run_delta<7, 2, 8, 2, 32, 3>(d32, bp, tmap, st, sh, sms);
        if (op == 1) return bp.csc ? run_check<7, 2, 32>(bp, st, sms) : run_check<7, 2, 64>(bp, st, sms);
        if (op == 2) return run_delta64<7, 2, 4, 2, 16, 4>(d64, bp, tmap, st, sh, sms);
        return cudaErrorNotSupported;
    }
    if (s == 3) {
        if (op == 0) return run_delta<7, 3, 4, 2, 16, 3>(d32, bp, tmap, st, sh, sms);
        if (op == 1) return bp.csc ? run_check<7, 3, 32>(bp, st, sms) : run_check<7, 3, 64>(bp, st, sms);
        if (op == 2) return run_delta64<7, 3, 4, 2, 16, 2>(d64, bp, tmap, st, sh, sms);
        return cudaErrorNotSupported;
    }
    return cudaErrorInvalidValue;
}

}  // namespace spb
