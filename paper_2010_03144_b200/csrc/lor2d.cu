// lor2d.cu -- Lorenzo blocks of 2-D fields (nx == 1, block edge 10: 1 x by x bz blocks) with a
// lane per block, compress (stage (c), pipeline.py:246-256,199-213) and decompress
// (_reconstruct_group, pipeline.py:586-638, with the sum_dc verification).
//
// With i == 0 the 7-term Lorenzo sum reduces to the (j - 1, k), (j, k - 1), (j - 1, k - 1)
// neighbours, evaluated here in the reference's 7-term order with the zero terms kept (their
// signed-zero effects stay bit-exact).  A lane walks its block row by row: the previous row's
// float64 reconstruction lives in registers, so a block needs no shared-memory buffer and no
// wavefront synchronisation, and a warp's 32 lanes (32 consecutive blocks along z) read and
// write their rows as contiguous 1280-byte runs.  The warp-per-block kernels (k_quant_lor,
// k_recon_g) keep 10-point planes on 10 of 32 lanes; here every lane works.
//
// Compress defers to k_quant_lor every block that carries injected faults or fails its stage (a)
// checksum (tile_correct's warp-wide search), through a second list.
namespace ftlz {

#define L2_E 10

// the reference's 7-term Lorenzo sum with i == 0 (d100 = d110 = d101 = d111 = 0)
FTLZ_DEV double lor2d_pred(double d010, double d001, double d011) {
    return __dadd_rn(__dadd_rn(__dadd_rn(__dadd_rn(__dadd_rn(__dadd_rn(0.0, d010), d001), -0.0), -0.0), -d011), 0.0);
}

__global__ void __launch_bounds__(128) k_quant_lor2d(CompArgs A) {
    if (dev_failed(A.st)) return;
    __shared__ u32 hwin[HWIN];
    const Geom& g = A.g;
    const int lane = threadIdx.x & 31;
    const int wlo = A.center - HWIN / 2;
    for (int t = threadIdx.x; t < HWIN; t += blockDim.x) hwin[t] = 0;
    __syncthreads();
    const QuantParams Q = *A.qp;
    const bool dup = A.dup_eval != 0;
    const u32 n = A.counters[4];
    const u32 nt = gridDim.x * blockDim.x;
    // whole warps iterate together (the histogram step is warp-collective)
    const u32 gtid = blockIdx.x * blockDim.x + threadIdx.x;
    for (u32 base_t = gtid - lane; base_t < n; base_t += nt) {
        const u32 t = base_t + lane;
        bool act = t < n;
        const long long b = act ? (long long)A.lor_list[t] : 0;
        if (act && (A.events[b] & 4)) act = false;
        BlockInfo B = block_info(g, b);
        const int by = B.by, bz = B.bz;
        // blocks with injected faults go to k_quant_lor
        if (act && A.n_faults && A.fault_first[b] >= 0) {
            A.defer_list[atomicAdd(&A.counters[9], 1u)] = (u32)b;
            act = false;
        }
        const float* xb = A.x + (B.bj * L2_E) * g.nz + B.bk * L2_E;
        // stage (a) verification: a mismatch (an SDC since k_prep) goes to tile_correct
        if (act && A.protect_input) {
            u64 s = 0, si = 0;
            for (int j = 0; j < by; j++)
                for (int k = 0; k < bz; k++) {
                    const u32 u = __float_as_uint(__ldg(xb + (long long)j * g.nz + k));
                    s += u;
                    si += (u64)(u32)(j * bz + k) * u;
                }
            if (s != A.insum[b] || si != A.inisum[b]) {
                A.defer_list[atomicAdd(&A.counters[9], 1u)] = (u32)b;
                act = false;
            }
        }
        u16* bins = A.bins + bins_index(g, b, 0);
        u32* unp = A.unp_scratch + (size_t)b * g.vmax;
        u64 bs = 0, bis = 0, dcsum = 0;
        u32 nunp = 0;
        bool mism = false;
        double prev[L2_E], cur[L2_E];
#pragma unroll
        for (int k = 0; k < L2_E; k++) prev[k] = 0.0;
        for (int j = 0; j < L2_E; j++) {
            const bool rowact = act && j < by;
            float xr[L2_E];
#pragma unroll
            for (int k = 0; k < L2_E; k++) xr[k] = (rowact && k < bz) ? __ldg(xb + (long long)j * g.nz + k) : 0.0f;
#pragma unroll
            for (int k = 0; k < L2_E; k++) {
                const bool on = rowact && k < bz;
                const double d010 = j > 0 ? prev[k] : 0.0;
                const double d001 = k > 0 ? cur[k > 0 ? k - 1 : 0] : 0.0;
                const double d011 = (j > 0 && k > 0) ? prev[k > 0 ? k - 1 : 0] : 0.0;
                const double p1 = lor2d_pred(d010, d001, d011);
                auto again = [&]() { return lor2d_pred(opaque(d010), opaque(d001), opaque(d011)); };
                DupMask M;
#pragma unroll
                for (int r = 0; r < 3; r++) M.p[r] = M.r[r] = 0ull;
                float r32;
                double back;
                const int bin = quant_point(Q, xr[k], p1, dup, again, again, M, &r32, &mism, &back);
                cur[k] = back;
                const int p = j * bz + k;
                if (on) {
                    bins[p] = (u16)bin;
                    bs += (u64)bin;
                    bis += (u64)p * (u64)bin;
                    dcsum += __float_as_uint(r32);
                    if (bin == 0) unp[nunp++] = __float_as_uint(xr[k]);
                }
                const unsigned peers = __match_any_sync(0xffffffffu, on ? bin : -1);
                if (on && lane == __ffs(peers) - 1) hist_add_w<HWIN>(hwin, A.hist, wlo, bin, (u32)__popc(peers));
            }
#pragma unroll
            for (int k = 0; k < L2_E; k++) prev[k] = cur[k];
        }
        if (act) {
            if (mism) atomicOr(&A.counters[1], 1u << (B.xid * 2 + 0));
            A.unpc[b] = nunp;
            if (nunp) atomicAdd((u64*)&A.layout[LAYOUT_NUNP], (u64)nunp);
            A.bsum[b] = bs;
            A.bisum[b] = bis;
            A.dcs[b] = dcsum;
        }
    }
    __syncthreads();
    hist_flush(hwin, A.hist, wlo, A.cap);
}

// decompress: Lorenzo blocks of 2-D fields, a lane per block, from the scratch bins of the
// decoder; unpredictable words in point order; decompressed-data faults applied; sum_dc verified
__global__ void __launch_bounds__(128) k_recon_lor2d(DecArgs A) {
    if (dev_failed(A.st)) return;
    const Geom& g = A.g;
    const u32 n = A.counters[DC_NLOR];
    const u32 gtid = blockIdx.x * blockDim.x + threadIdx.x;
    for (u32 t = gtid; t < n; t += gridDim.x * blockDim.x) {
        const long long b = A.lor_list[t];
        if (b < A.sb0 || b >= A.sb1) continue;   // another slab's block
        if (A.dflag[b]) continue;                 // undecodable: reported separately
        const BlockInfo B = block_info(g, b);
        const int by = B.by, bz = B.bz;
        const u16* bins = A.bins + bins_index(g, b, 0);
        const u64 unp_base = A.info[DI_UNP_OFF] + 4 * A.uofs[b];
        const int f0 = A.n_faults ? A.fault_first[b] : -1;
        float* ob = A.out + (B.bj * L2_E) * g.nz + B.bk * L2_E;
        u32 zeros = 0;
        u64 dsum = 0;
        double prev[L2_E], cur[L2_E];
#pragma unroll
        for (int k = 0; k < L2_E; k++) prev[k] = 0.0;
        for (int j = 0; j < by; j++) {
#pragma unroll
            for (int k = 0; k < L2_E; k++) {
                if (k < bz) {
                    const int p = j * bz + k;
                    const u32 bin = bins[p];
                    const double d010 = j > 0 ? prev[k] : 0.0;
                    const double d001 = k > 0 ? cur[k > 0 ? k - 1 : 0] : 0.0;
                    const double d011 = (j > 0 && k > 0) ? prev[k > 0 ? k - 1 : 0] : 0.0;
                    float v;
                    if (bin) {
                        const double pred = lor2d_pred(d010, d001, d011);
                        v = __double2float_rn(__dadd_rn(pred, __dmul_rn(A.twoeb, int_to_f64((int)bin - A.center))));
                    } else {
                        v = __uint_as_float((u32)ld_le(A.a + unp_base + 4ull * zeros, 4));
                        zeros++;
                    }
                    cur[k] = f32_to_f64(v);
                    if (f0 >= 0) v = apply_decomp_faults(A, b, p, f0, v);
                    dsum += __float_as_uint(v);
                    ob[(long long)j * g.nz + k] = v;
                }
            }
#pragma unroll
            for (int k = 0; k < L2_E; k++) prev[k] = cur[k];
        }
        if (A.info[DI_HAS_SDC] && stored_sum_dc(A, b) != dsum) {
            A.mflag[b] = 1;
            A.mis_list[atomicAdd(&A.counters[DC_NMIS], 1u)] = (u32)b;
        }
    }
}

}  // namespace ftlz
