// Measured and not adopted (profiles/r6/r6o_ab.txt: conv3 forward 24.4k vs 25.6k cycles per iteration, 4.260 M vs
// 4.254 M samples/s, within noise; 20 lanes per warp: 4.17 M).  Parity-green on the large-net subset.  Kept for the record.
// ------------------------------------------------------------------------------------
// PHASE(conv_fwd_bm) conv -> tanh -> max-pool forward of a SMALL input (the large net's conv3: 60 maps
// of 5x5 -> 100 maps, 2x2 kernel, 2x2 pool) with the lanes over OUTPUT maps and the input as
// warp-uniform 16-byte broadcast loads.  A warp task = (image, block of ML maps); lane l owns map
// mb * ML + l and all OH x OW conv outputs of the image.  Four input maps at a time: their 4 H W
// contiguous floats arrive as H W uniform 16-byte loads (2 shared-memory wavefronts each for the whole
// warp) and every word is multiplied into the <= K*K outputs it reaches with the lane's own weights
// (conflict-free scalar loads: maps are the fastest index of the staged W).  conv_fwd's items load a
// private 3x3 patch and a 16-byte weight vector per tap (non-uniform: 4 wavefronts): 25 wavefronts per
// 16 FMA-pipe cycles per input map and warp, with 400 items on 640 threads; here 10 wavefronts per 16.
// Horizontally adjacent outputs share one packed FMA where their accumulator pair is even-aligned.
// Every accumulator sums bias, then (n, i, j) ascending: bitwise conv_fwd's values.
// ------------------------------------------------------------------------------------
template <class L, int NT, int ML>
__device__ __forceinline__ void conv_fwd_bm(const float* __restrict__ in, const float* __restrict__ wsm,
                                            float* __restrict__ out, uint8_t* __restrict__ am, int cnt) {
    constexpr int K = L::K, KP = L::KP, H = L::H, W = L::W, HW = H * W, OH = L::OH, OW = L::OW;
    constexpr int PH = L::PH, PW = L::PW, P = L::P, M = L::M, C = L::C;
    constexpr int NB = 4, NV = NB * HW / 4, MB = M / ML, NW = NT / 32;
    static_assert(K == 2 && KP == 2 && OH == PH * KP && OW == PW * KP && OW % 2 == 0, "2x2 kernel, 2x2 pool, no dropped rows");
    static_assert(C % NB == 0 && (NB * HW) % 4 == 0 && L::IN_SZ % 4 == 0, "16-byte blocks of 4 input maps");
    static_assert(M % ML == 0 && ML <= 32, "ML lanes, one map each");
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const bool act = lane < ML;
    for (int task = warp; task < cnt * MB; task += NW) {
        const int mb = task % MB, g = task / MB;
        const int m = mb * ML + (act ? lane : 0);
        float acc[OH][OW];
        {
            const float b = wsm[L::WFL + m];
#pragma unroll
            for (int y = 0; y < OH; ++y)
#pragma unroll
                for (int x = 0; x < OW; ++x) acc[y][x] = b;
        }
        const float4* ib = reinterpret_cast<const float4*>(in + g * L::IN_SZ);
#pragma unroll 1
        for (int n0 = 0; n0 < C; n0 += NB) {
            // the lane's weights of the 4 maps, each tap row as the reversed pair (w[i][1], w[i][0]): the
            // word at column x feeds output x - 1 through tap column 1 and output x through tap column 0
            float wr[NB][K][2];
#pragma unroll
            for (int nn = 0; nn < NB; ++nn)
#pragma unroll
                for (int i = 0; i < K; ++i) {
                    wr[nn][i][0] = wsm[(n0 + nn) * L::NS + (i * K + 1) * L::MP + m];
                    wr[nn][i][1] = wsm[(n0 + nn) * L::NS + (i * K) * L::MP + m];
                }
#pragma unroll
            for (int v = 0; v < NV; ++v) {
                const float4 xv = ib[n0 * HW / 4 + v];  // warp-uniform
                const float xs[4] = {xv.x, xv.y, xv.z, xv.w};
#pragma unroll
                for (int e = 0; e < 4; ++e) {
                    const int idx = v * 4 + e, nn = idx / HW, y = (idx % HW) / W, x = idx % W;
#pragma unroll
                    for (int i = 0; i < K; ++i) {
                        const int oy = y - i;
                        if (oy < 0 || oy >= OH) continue;  // compile-time after unrolling
                        if (x >= 1 && x < OW && (x - 1) % 2 == 0 && (L::FF & 1)) {
                            fma_pair(acc[oy][x - 1], acc[oy][x], wr[nn][i][0], wr[nn][i][1], xs[e]);
                        } else {
                            if (x < OW) acc[oy][x] = fmaf(wr[nn][i][1], xs[e], acc[oy][x]);            // j = 0
                            if (x >= 1) acc[oy][x - 1] = fmaf(wr[nn][i][0], xs[e], acc[oy][x - 1]);  // j = 1
                        }
                    }
                }
            }
        }
        if (act) {
#pragma unroll
            for (int pr = 0; pr < PH; ++pr)
#pragma unroll
                for (int pc = 0; pc < PW; ++pc) {
                    float best = acc[pr * KP][pc * KP];
                    int arg = 0;
#pragma unroll
                    for (int q = 1; q < KP * KP; ++q) {
                        const float vq = acc[pr * KP + q / KP][pc * KP + q % KP];
                        if (vq > best) {  // first strict maximum wins (R4)
                            best = vq;
                            arg = q;
                        }
                    }
                    const int o = g * L::OUT_SZ + m * P + pr * PW + pc;
                    out[o] = tanhf(best);
                    am[o] = static_cast<uint8_t>(arg);
                }
        }
    }
}

