// Measured and not adopted (profiles/r6/r6h_ab.txt: 4.186 M vs 4.254 M samples/s; conv2 forward 51.9k vs 48.1k
// cycles per iteration).  Parity-green on the large-net subset.  Kept here for the record only.
// ------------------------------------------------------------------------------------
// PHASE(conv_fwd_lm) conv -> tanh -> max-pool forward with the LANES OVER OUTPUT MAPS (KP == 2).
// A warp task = (image, window row, block of 2 * ML maps); lane l owns the maps mb + l and mb + ML + l
// and their KP conv rows x 2 PW conv columns of the window row (2 x KP x 2 PW accumulators).  Per
// input map the KP + K - 1 input rows the window row reads are loaded once each as warp-uniform
// scalars (broadcast: one shared-memory wavefront per word for the whole warp) and the lane's own
// K*K weights of its two maps as conflict-free scalar loads (maps are the fastest index of the staged
// W), so a word loaded feeds 2 x 2 PW / (2 PW + K - 1) x K FMAs and the FMA pipe, not the shared-memory
// wavefront rate, bounds the loop (conv_fwd's weight vectors over map groups cost their full width:
// 106 wavefronts per 90 FMA-pipe cycles on the large net's conv2).  The two maps of a lane share one
// packed FMA (fma_pair).  Every accumulator sums bias, then (n, i, j) ascending: bitwise conv_fwd's
// values.
// ------------------------------------------------------------------------------------
template <class L, int NT, int ML>
__device__ __forceinline__ void conv_fwd_lm(const float* __restrict__ in, const float* __restrict__ wsm,
                                            float* __restrict__ out, uint8_t* __restrict__ am, int cnt) {
    constexpr int K = L::K, KP = L::KP, PW = L::PW, PH = L::PH, P = L::P, M = L::M, C = L::C;
    constexpr int CW = KP * PW, RL = CW + K - 1, PR = KP + K - 1;  // conv columns, input row words, input rows
    constexpr int MB = M / (2 * ML), NW = NT / 32;
    static_assert(KP == 2 && M % (2 * ML) == 0 && ML <= 32, "2x2 pooling, 2 maps per lane");
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const bool act = lane < ML;
    for (int task = warp; task < cnt * PH * MB; task += NW) {
        const int mb = task % MB, pr = (task / MB) % PH, g = task / (MB * PH);
        const int m0 = mb * 2 * ML + (act ? lane : 0), m1 = m0 + ML;
        float acc[KP][CW][2];
        {
            const float b0 = wsm[L::WFL + m0], b1 = wsm[L::WFL + m1];
#pragma unroll
            for (int u = 0; u < KP; ++u)
#pragma unroll
                for (int c = 0; c < CW; ++c) {
                    acc[u][c][0] = b0;
                    acc[u][c][1] = b1;
                }
        }
        const float* ib = in + g * L::IN_SZ + (pr * KP) * L::W;
#pragma unroll 1
        for (int n = 0; n < C; ++n) {
            float w[K * K][2];
#pragma unroll
            for (int t = 0; t < K * K; ++t) {
                w[t][0] = wsm[n * L::NS + t * L::MP + m0];
                w[t][1] = wsm[n * L::NS + t * L::MP + m1];
            }
            const float* ir = ib + n * (L::H * L::W);
#pragma unroll
            for (int r = 0; r < PR; ++r) {
                float x[RL];
#pragma unroll
                for (int c = 0; c < RL; ++c) x[c] = ir[r * L::W + c];  // warp-uniform
#pragma unroll
                for (int u = 0; u < KP; ++u) {
                    const int i = r - u;  // tap row of conv row u that reads input row r
                    if (i >= 0 && i < K) {
#pragma unroll
                        for (int j = 0; j < K; ++j)
#pragma unroll
                            for (int c = 0; c < CW; ++c)
                                fma_pair(acc[u][c][0], acc[u][c][1], w[i * K + j][0], w[i * K + j][1], x[c + j]);
                    }
                }
            }
        }
        if (act) {
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                const int m = h == 0 ? m0 : m1;
#pragma unroll
                for (int pc = 0; pc < PW; ++pc) {
                    float best = acc[0][pc * KP][h];
                    int arg = 0;
#pragma unroll
                    for (int q = 1; q < KP * KP; ++q) {
                        const float v = acc[q / KP][pc * KP + q % KP][h];
                        if (v > best) {  // first strict maximum wins (R4)
                            best = v;
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
}

