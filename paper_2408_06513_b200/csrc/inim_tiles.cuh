// Tile reduce (phase 1 of the integral pass), shared by the standalone reduce kernel
// (integral.cu) and the fused smoothing kernel (smooth.cu).
//
// One thread group of NW*32 threads owns one TH x TW tile held in shared memory
// (row stride TW); lane u of warp w owns column 32*w + u and sweeps the TH rows.
// Emitted per tile (all band-local, no inter-tile dependency):
//   colsum[b][c]   column sums of the tile (= in-band column prefix V at the last row)
//   rowsum[j][x]   row sums of the tile
//   ulbot[b][c]    in-tile up-left chain of V at the band's last row
//   urbot[b][c]    in-tile up-right chain of V at the band's last row
//   ule[b][x][r]   up-left chain at the tile's last column (complete in-band value)
//   ure[b][x][r]   up-right chain at the tile's first column (complete in-band value)
#pragma once

#include "inim_internal.cuh"

namespace inim {

// rec: 3 * NW * TH floats of shared scratch for this group.  tid: thread index within
// the group.  All groups of the CTA must call this together (one __syncthreads inside).
__device__ __forceinline__ void tile_reduce(const float* sd, float* rec, const Geo g, const Ws ws, int b, int x,
                                            int tid) {
    const int lane = tid & 31, w = tid >> 5;
    const int TH = g.TH, TW = g.TW, NW = g.NW, WL = g.WL, s = g.s, NX = g.NX;
    const int u = w * 32 + lane;
    const bool act = u < TW;
    const int edge = WL - 1;
    float* ULR = rec;
    float* URL = rec + NW * TH;
    float* RS = rec + 2 * NW * TH;

    float V = 0.f, ULw = 0.f, URw = 0.f;
    for (int r = 0; r < TH; ++r) {
        const float dv = act ? sd[r * TW + u] : 0.f;
        V += dv;
        const float upUL = __shfl_up_sync(kFull, ULw, 1);
        const float dnUR = __shfl_down_sync(kFull, URw, 1);
        ULw = V + (lane > 0 ? upUL : 0.f);
        URw = V + (lane < 31 ? dnUR : 0.f);
        const float rs = warp_sum(dv);
        if (lane == edge) ULR[w * TH + r] = ULw;
        if (lane == 0) {
            URL[w * TH + r] = URw;
            RS[w * TH + r] = rs;
        }
    }
    __syncthreads();

    const int a = b * TH, i0 = x * TW;
    const int64_t tile = (int64_t)b * NX + x;
    if (act) {
        ws.colsum[(int64_t)b * s + i0 + u] = V;
        float ulb = ULw, urb = URw;
        const int rr = TH - 2 - lane;  // row where the up-left chain from the last row leaves this warp
        if (w > 0 && rr >= 0) ulb += ULR[(w - 1) * TH + rr];
        const int rq = TH - 1 - (WL - lane);  // row where the up-right chain leaves this warp
        if (w < NW - 1 && rq >= 0) urb += URL[(w + 1) * TH + rq];
        ws.ulbot[(int64_t)b * s + i0 + u] = ulb;
        ws.urbot[(int64_t)b * s + i0 + u] = urb;
    }
    if (tid < TH) {
        const int r = tid;
        ws.ule[tile * TH + r] = ULR[(NW - 1) * TH + r];
        ws.ure[tile * TH + r] = URL[r];
        float rs = 0.f;
        for (int ww = 0; ww < NW; ++ww) rs += RS[ww * TH + r];
        ws.rowsum[(int64_t)(a + r) * NX + x] = rs;
    }
}

}  // namespace inim
