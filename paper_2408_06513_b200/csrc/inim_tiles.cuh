// Tile reduce (phase 1 of the integral pass), shared by the standalone reduce kernel
// (integral.cu) and the fused smoothing kernel (smooth.cu).
#pragma once

#include "inim_internal.cuh"

namespace inim {

// =====================================================================================
// Tile reduce (phase 1).  sd: TH x TW tile of d in shared memory (row stride TW).
// rec: 5 * NW * TH floats of shared scratch.  blockDim.x == NW * 32.
// =====================================================================================
__device__ __forceinline__ void tile_reduce(const float* sd, float* rec, const Geo g, const Ws ws, int b, int x) {
    const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
    const int TH = g.TH, TW = g.TW, NW = g.NW, WL = g.WL, s = g.s, NX = g.NX;
    const int u = w * 32 + lane;
    const bool act = u < TW;
    const int edge = WL - 1;
    float* ULR = rec;
    float* URL = rec + NW * TH;
    float* DDR = rec + 2 * NW * TH;
    float* ADL = rec + 3 * NW * TH;
    float* RS = rec + 4 * NW * TH;

    float V = 0.f, ULw = 0.f, URw = 0.f, dd = 0.f, ad = 0.f;
    for (int r = 0; r < TH; ++r) {
        const float dv = act ? sd[r * TW + u] : 0.f;
        V += dv;
        const float upUL = __shfl_up_sync(kFull, ULw, 1);
        const float upDD = __shfl_up_sync(kFull, dd, 1);
        const float dnUR = __shfl_down_sync(kFull, URw, 1);
        const float dnAD = __shfl_down_sync(kFull, ad, 1);
        ULw = V + (lane > 0 ? upUL : 0.f);
        dd = dv + (lane > 0 ? upDD : 0.f);
        URw = V + (lane < 31 ? dnUR : 0.f);
        ad = dv + (lane < 31 ? dnAD : 0.f);
        const float rs = warp_sum(dv);
        if (lane == edge) {
            ULR[w * TH + r] = ULw;
            DDR[w * TH + r] = dd;
        }
        if (lane == 0) {
            URL[w * TH + r] = URw;
            ADL[w * TH + r] = ad;
            RS[w * TH + r] = rs;
        }
    }
    __syncthreads();

    const int a = b * TH, i0 = x * TW;
    const int ND = TW + TH - 1;
    const int64_t tile = (int64_t)b * NX + x;
    float* dp = ws.dpart + tile * ND;
    float* ap = ws.apart + tile * ND;
    if (act) {
        ws.colsum[(int64_t)b * s + i0 + u] = V;
        float ulb = ULw, ddb = dd, urb = URw, adb = ad;
        const int rr = TH - 2 - lane;  // row where the up-left chain from the last row leaves this warp
        if (w > 0 && rr >= 0) {
            ulb += ULR[(w - 1) * TH + rr];
            ddb += DDR[(w - 1) * TH + rr];
        }
        const int rq = TH - 1 - (WL - lane);  // row where the up-right chain leaves this warp
        if (w < NW - 1 && rq >= 0) {
            urb += URL[(w + 1) * TH + rq];
            adb += ADL[(w + 1) * TH + rq];
        }
        ws.ulbot[(int64_t)b * s + i0 + u] = ulb;
        ws.urbot[(int64_t)b * s + i0 + u] = urb;
        dp[u] = ddb;            // diagonal t = u ends on the last row
        ap[u + TH - 1] = adb;   // anti-diagonal t = u + TH - 1 ends on the last row
    }
    if (tid < TH) {
        const int r = tid;
        if (r < TH - 1) {
            dp[TW + TH - 2 - r] = DDR[(NW - 1) * TH + r];  // diagonals leaving through the right edge
            ap[r] = ADL[r];                                 // anti-diagonals leaving through the left edge
        }
        ws.ule[tile * TH + r] = ULR[(NW - 1) * TH + r];
        ws.ure[tile * TH + r] = URL[r];
        float rs = 0.f;
        for (int ww = 0; ww < NW; ++ww) rs += RS[ww * TH + r];
        ws.rowsum[(int64_t)(a + r) * NX + x] = rs;
    }
}

}  // namespace inim
