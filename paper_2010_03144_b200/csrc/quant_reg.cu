// quant_reg.cu -- stage (c) of pipeline.compress for regression blocks (pipeline.py:390-409,
// 442-453): verify input, predict (duplicated), quantize, reconstruct (duplicated),
// double-check, bins / unpredictable words / checksums / sum_dc / histogram.
//
// Persistent CTAs walk "pencils" (P blocks along z, blocks.cu) with a two-stage cp.async
// pipeline; inside a pencil one thread owns one row (i, j) of one block.  The hot loop over a
// row is branch-free: every point takes the fast quantizer (reciprocal multiply, 2^52-magic
// floor) and raises a flag when it lies within a few ulps of a decision threshold, when the
// duplicated evaluations disagree, or when the bound forces exact division.  A flagged row is
// recomputed with the exact reference formulation (blocks.cu quant_point), so the fast path
// never changes a result.  The input checksum (stage (a) pair from k_prep) is accumulated in
// the same loop and verified afterwards; a mismatching block is corrected
// (checksum.py:109-142) and recomputed.  Partial sums are reduced per block by one warp
// (64-bit shared atomics would compile to CAS loops on sm_100).
namespace ftlz {

// quantize() contract (common.cuh) without branches; `slow` is raised instead of resolving
// an ambiguous point.  floor(fl(h + 0.5)) = RN(t) - (t < RN(t)) with RN(t) from t + 2^52
// and the exact residual d = t - RN(t); |d| < 2^-30 means t sits at an integer, where the
// reciprocal's <= 3 ulp error could change the floor.
FTLZ_DEV int quant_fast(double h_rcp, double diff, const QuantParams& Q, bool& ok, u32& slow) {
    double h = __dmul_rn(fabs(diff), h_rcp);
    u64 hb = dbits(h);
    bool small = hb <= Q.capd2_bits;
    slow |= ((u32)(hb >> 32) - (u32)(Q.capd2_bits >> 32) + 1u) < 2u;  // h' within 2^-20 rel of 2*cap
    double t = __dadd_rn(h, 0.5);
    double m = __dadd_rn(t, 4503599627370496.0);   // 2^52: low word = RN(t)
    double r = __dadd_rn(m, -4503599627370496.0);
    double d = __dadd_rn(t, -r);                   // exact (Sterbenz)
    u32 dhi = (u32)(dbits(d) >> 32);
    int q = (int)(u32)dbits(m) - (int)(dhi >> 31);
    slow |= (u32)(small && ((dhi & 0x7fffffffu) < 0x3e100000u));
    q = small ? q : 0;
    int s = (int)(u32)(dbits(diff) >> 32) >> 31;   // 0 or -1
    q = (q ^ s) - s;
    int b = Q.center + q;
    ok = small && (u32)(b - 1) < (u32)(Q.cap - 1);
    return ok ? b : 0;
}

struct RowAcc {
    u64 cs, csi, bis, dc;
    u32 bs, nz;
};

// exact recomputation of one row (reference operand order, 2-of-3 voting on mismatch)
FTLZ_DEV void row_exact(const QuantParams& Q, const float* xr, int bz, int p0, double ab, double ab2,
                        const double* ctab, float4 cf, int i, int j, bool dup, u16* bins16, RowAcc& acc,
                        bool& mism) {
    double c0 = (double)cf.x, c1 = (double)cf.y, c2 = (double)cf.z, c3 = (double)cf.w;
    acc.bis = 0;
    acc.dc = 0;
    acc.bs = 0;
    acc.nz = 0;
    for (int k = 0; k < bz; k++) {
        double ck = ctab[k];
        double p1 = __dadd_rn(ab, ck), p2 = __dadd_rn(ab2, ck);
        float r32;
        double back;
        int bin = quant_point<>(Q, xr[k], p1, p2, dup,
                                [&] {
                                    return __dadd_rn(__dadd_rn(__dadd_rn(c0, __dmul_rn(c1, int_to_f64(i))), __dmul_rn(c2, int_to_f64(j))),
                                                     __dmul_rn(c3, int_to_f64(k)));
                                },
                                &r32, &mism, &back);
        bins16[k] = (u16)bin;
        acc.bs += (u32)bin;
        acc.bis += (u64)(u32)(p0 + k) * (u64)(u32)bin;
        acc.dc += __float_as_uint(r32);
        acc.nz += bin == 0;
    }
}

// fast row: returns nonzero when the row must be recomputed exactly
template <bool DUP, bool PIN, int BZ>
FTLZ_DEV u32 row_fast(const QuantParams& Q, const float* xr, int bz_rt, u32 p0, double ab, double ab2,
                      const double* ctab, u16* bins16, RowAcc& acc) {
    const int bz = BZ > 0 ? BZ : bz_rt;
    u32 slow = (u32)Q.exact_div;
    u32 dm = 0;
    const double rcp = Q.rcp, twoeb = Q.twoeb, twoeb2 = Q.twoeb_dup, eb = Q.eb;
    // even compile-time rows: 8-byte loads of x and 4-byte stores of bin pairs (half the shared
    // memory instructions; rows start 8-byte aligned since stride and e are even)
    constexpr bool PAIRS = BZ > 0 && (BZ % 2) == 0;
    float xs[PAIRS ? BZ : 1];
    u32 lo_bin = 0;
    if constexpr (PAIRS) {
#pragma unroll
        for (int k = 0; k < BZ; k += 2) {
            float2 v = *(const float2*)(xr + k);
            xs[k] = v.x;
            xs[k + 1] = v.y;
        }
    }
    auto point = [&](int k) {
        float x32;
        if constexpr (PAIRS) x32 = xs[k];
        else x32 = xr[k];
        u32 u = __float_as_uint(x32);
        u32 p = p0 + (u32)k;
        if (PIN) {
            acc.cs += (u64)u;
            acc.csi += (u64)p * (u64)u;
        }
        double x64 = (double)x32;
        double ck = ctab[k];
        double p1 = __dadd_rn(ab, ck);
        bool ok;
        int bin = quant_fast(rcp, __dadd_rn(x64, -p1), Q, ok, slow);
        double offs = int_to_f64(ok ? bin - Q.center : -Q.center);
        double d1 = __dadd_rn(p1, __dmul_rn(twoeb, offs));
        if (DUP) {
            // second evaluation from independently loaded operands (ab2, twoeb2)
            double p2 = __dadd_rn(ab2, ck);
            double d2 = __dadd_rn(p2, __dmul_rn(twoeb2, offs));
            u64 x = (dbits(p1) ^ dbits(p2)) | (dbits(d1) ^ dbits(d2));
            dm |= (u32)x | (u32)(x >> 32);
        }
        float d32 = __double2float_rn(d1);
        bool keep = ok && fabs(__dadd_rn(x64, -(double)d32)) <= eb;
        u32 fb = keep ? (u32)bin : 0u;
        float r32 = keep ? d32 : x32;
        if constexpr (PAIRS) {
            if (k & 1) *(u32*)(bins16 + k - 1) = lo_bin | (fb << 16);
            else lo_bin = fb;
        } else {
            bins16[k] = (u16)fb;
        }
        acc.bs += fb;
        acc.bis += (u64)p * (u64)fb;
        acc.dc += (u64)__float_as_uint(r32);
        acc.nz += fb == 0u;
    };
    if constexpr (BZ > 0) {
#pragma unroll
        for (int k = 0; k < BZ; k++) point(k);
    } else {
        for (int k = 0; k < bz; k++) point(k);
    }
    return slow | dm;
}

FTLZ_DEV float4 ld_volatile_f4(const float4* p) {
    float4 v;
    asm volatile("ld.volatile.global.v4.f32 {%0,%1,%2,%3}, [%4];"
                 : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
                 : "l"(p));
    return v;
}

__global__ void __launch_bounds__(416, 2) k_quant_reg(CompArgs A) {
    extern __shared__ __align__(16) unsigned char smem[];
    const Geom& g = A.g;
    if (dev_failed(A.st)) return;
    int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31, nthr = blockDim.x;
    const int nv8 = g.nvmax8;
    const size_t tb = (size_t)A.tile_bytes;
    u16* bins_all = (u16*)(smem + 2 * tb);
    double* ctab_all = (double*)(smem + 2 * tb + (((size_t)2 * nv8 * A.P + 15) & ~(size_t)15));
    u32* hwin = (u32*)(ctab_all + 64 * A.P);
    RowAcc* racc = (RowAcc*)(hwin + HWIN);   // per-row partial sums
    const int wlo = A.center - HWIN / 2;
    for (int t = tid; t < HWIN; t += nthr) hwin[t] = 0;
    __shared__ int s_any, s_kind[16];
    __shared__ u64 s_cs[16], s_csi[16], s_bis[16], s_dc[16];
    __shared__ u32 s_bs[16], s_nz[16];
    const QuantParams Q = *A.qp;
    const bool dup = A.dup_eval != 0, pin = A.protect_input != 0;
    auto reduce_block = [&](int wb, int rows) {
        RowAcc t = {0, 0, 0, 0, 0, 0};
        for (int r = lane; r < rows; r += 32) {
            const RowAcc& a = racc[wb * rows + r];
            t.cs += a.cs; t.csi += a.csi; t.bis += a.bis; t.dc += a.dc; t.bs += a.bs; t.nz += a.nz;
        }
        t.cs = warp_sum_u64(t.cs); t.csi = warp_sum_u64(t.csi);
        t.bis = warp_sum_u64(t.bis); t.dc = warp_sum_u64(t.dc);
        t.bs = warp_sum_u32(t.bs); t.nz = warp_sum_u32(t.nz);
        if (lane == 0) {
            s_cs[wb] = t.cs; s_csi[wb] = t.csi; s_bis[wb] = t.bis; s_dc[wb] = t.dc;
            s_bs[wb] = t.bs; s_nz[wb] = t.nz;
        }
    };
    long long np = A.npencils, G = gridDim.x;
    long long pid = blockIdx.x;
    if (pid < np) {
        Pencil P0 = pencil_of(g, (u32)pid, A.P, A.fd_npz, A.fd_cy);
        issue_pencil(A.x, g, P0, (float*)smem, A.tile_stride, P0.by == g.e ? A.fd_e : A.fd_ry, A.pio, A.P);
    }
    cp_commit();
    int buf = 0;
    for (; pid < np; pid += G) {
        if (pid + G < np) {
            Pencil P1 = pencil_of(g, (u32)(pid + G), A.P, A.fd_npz, A.fd_cy);
            issue_pencil(A.x, g, P1, (float*)(smem + (buf ^ 1) * tb), A.tile_stride, P1.by == g.e ? A.fd_e : A.fd_ry, A.pio, A.P);
        }
        cp_commit();
        Pencil Pn = pencil_of(g, (u32)pid, A.P, A.fd_npz, A.fd_cy);
        float* tile = (float*)(smem + buf * tb);
        long long b0 = ((Pn.bi * g.cy) + Pn.bj) * g.cz + Pn.bk0;
        // per-block setup while the tile is still streaming in
        if (warp < Pn.nblk) {
            int k = A.ind[b0 + warp];
            if (A.events[b0 + warp] & 4) k = 2;  // stage (b) already failed this block
            if (lane == 0) s_kind[warp] = k;
            if (k == 1) {
                // C[k] = b3 * k (exact products, reference operand)
                double c3 = (double)A.coef[b0 + warp].w;
                for (int t = lane; t < 64; t += 32) ctab_all[warp * 64 + t] = __dmul_rn(c3, int_to_f64(t));
            }
        }
        if (tid == 0) s_any = 0;
        cp_wait1();
        __syncthreads();
        if (tid < Pn.nblk && s_kind[tid] == 1) s_any = 1;
        // working-array faults persist only without input protection (pipeline.py:331-361)
        if (!A.protect_input && A.n_faults && warp < Pn.nblk && s_kind[warp] == 1) {
            int bz = (warp == Pn.nblk - 1) ? Pn.bz_last : g.e;
            TileWalk w0;
            w0.bx = Pn.bx; w0.by = Pn.by; w0.bz = bz; w0.stride = A.tile_stride; w0.zoff = warp * g.e;
            apply_input_faults(A, b0 + warp, tile, w0, lane);
        }
        __syncthreads();
        if (s_any) {
            const int rows = Pn.bx * Pn.by;
            auto do_row = [&](int w, int r, bool exact) {
                long long b = b0 + w;
                int bz = (w == Pn.nblk - 1) ? Pn.bz_last : g.e;
                int i = (int)fdiv((u32)r, Pn.by == g.e ? A.fd_e : A.fd_ry), j = r - i * Pn.by;
                float4 cf = A.coef[b];
                double c0 = (double)cf.x, c1 = (double)cf.y, c2 = (double)cf.z;
                double di = int_to_f64(i), dj = int_to_f64(j);
                double ab = __dadd_rn(__dadd_rn(c0, __dmul_rn(c1, di)), __dmul_rn(c2, dj));
                double ab2 = ab;
                if (dup) {
                    float4 cg = ld_volatile_f4(A.coef + b);  // independent operands for eval 2
                    ab2 = __dadd_rn(__dadd_rn((double)cg.x, __dmul_rn((double)cg.y, di)), __dmul_rn((double)cg.z, dj));
                }
                const float* xr = tile + r * A.tile_stride + w * g.e;
                u16* bins16 = bins_all + (size_t)w * nv8 + (size_t)r * bz;
                const double* ctab = ctab_all + w * 64;
                u32 p0 = (u32)(r * bz);
                RowAcc acc = {0, 0, 0, 0, 0, 0};
                bool mism = false;
                u32 slow = exact;
                if (!exact) {
                    if (bz == 10) {
                        if (dup) slow = pin ? row_fast<true, true, 10>(Q, xr, bz, p0, ab, ab2, ctab, bins16, acc)
                                            : row_fast<true, false, 10>(Q, xr, bz, p0, ab, ab2, ctab, bins16, acc);
                        else slow = pin ? row_fast<false, true, 10>(Q, xr, bz, p0, ab, ab2, ctab, bins16, acc)
                                        : row_fast<false, false, 10>(Q, xr, bz, p0, ab, ab2, ctab, bins16, acc);
                    } else {
                        if (dup) slow = pin ? row_fast<true, true, 0>(Q, xr, bz, p0, ab, ab2, ctab, bins16, acc)
                                            : row_fast<true, false, 0>(Q, xr, bz, p0, ab, ab2, ctab, bins16, acc);
                        else slow = pin ? row_fast<false, true, 0>(Q, xr, bz, p0, ab, ab2, ctab, bins16, acc)
                                        : row_fast<false, false, 0>(Q, xr, bz, p0, ab, ab2, ctab, bins16, acc);
                    }
                } else {
                    for (int k = 0; k < bz; k++) {
                        u32 u = __float_as_uint(xr[k]);
                        acc.cs += u;
                        acc.csi += (u64)(p0 + k) * u;
                    }
                }
                if (slow) row_exact(Q, xr, bz, (int)p0, ab, ab2, ctab, cf, i, j, dup, bins16, acc, mism);
                racc[w * rows + r] = acc;
                if (mism) {
                    int xid = ((Pn.bx != g.e) ? 4 : 0) | ((Pn.by != g.e) ? 2 : 0) | ((bz != g.e) ? 1 : 0);
                    atomicOr(&A.counters[1], 1u << (xid * 2 + 1));
                }
            };
            for (int t = tid; t < rows * Pn.nblk; t += nthr) {
                int w = t / rows, r = t - (t / rows) * rows;
                if (s_kind[w] == 1) do_row(w, r, false);
            }
            __syncthreads();
            for (int wb = warp; wb < Pn.nblk; wb += nthr >> 5) {
                if (s_kind[wb] != 1) continue;
                reduce_block(wb, rows);
                __syncwarp();
                // stage (c) verification of the re-read input against the stage (a) pair
                long long b = b0 + wb;
                if (pin && (s_cs[wb] != A.insum[b] || s_csi[wb] != A.inisum[b])) {
                    int bz = (wb == Pn.nblk - 1) ? Pn.bz_last : g.e;
                    TileWalk w0;
                    w0.bx = Pn.bx; w0.by = Pn.by; w0.bz = bz; w0.stride = A.tile_stride; w0.zoff = wb * g.e;
                    int rr = tile_correct(tile, w0, rows * bz, A.insum[b], A.inisum[b], lane);
                    if (lane == 0) {
                        atomicAdd(&A.counters[3], 1u);
                        if (rr == 1) A.events[b] |= 1;
                        else { A.events[b] |= 4; s_kind[wb] = 2; }
                    }
                    __syncwarp();
                    if (rr == 1) {
                        for (int r = lane; r < rows; r += 32) do_row(wb, r, true);
                        __syncwarp();
                        reduce_block(wb, rows);
                    }
                    __syncwarp();
                }
                if (lane == 0 && s_kind[wb] == 1) {
                    A.unpc[b] = s_nz[wb];
                    if (s_nz[wb]) atomicAdd((u64*)&A.layout[LAYOUT_NUNP], (u64)s_nz[wb]);
                    A.bsum[b] = s_bs[wb];
                    A.bisum[b] = s_bis[wb];
                    A.dcs[b] = s_dc[wb];
                }
            }
            __syncthreads();
            // final bins: encoder layout (16-byte chunks), warp-aggregated histogram, and the
            // unpredictable words (rare) -- every warp takes a share of every block
            const int nch = (rows * g.e + 7) >> 3;
            for (int t = tid; t < Pn.nblk * nch; t += nthr) {
                int wb = t / nch, c = t - (t / nch) * nch;
                int bz = (wb == Pn.nblk - 1) ? Pn.bz_last : g.e;
                if (s_kind[wb] != 1 || 8 * c >= rows * bz) continue;
                *(uint4*)(A.bins + bins_index(g, b0 + wb, 8 * c)) = *(const uint4*)(bins_all + (size_t)wb * nv8 + 8 * c);
            }
            for (int wb = 0; wb < Pn.nblk; wb++) {
                if (s_kind[wb] != 1) continue;
                int vol = rows * ((wb == Pn.nblk - 1) ? Pn.bz_last : g.e);
                const u16* bins16 = bins_all + (size_t)wb * nv8;
                // two bins per lane (slots are 8-aligned); lanes holding the same bin add once
                for (int p0 = warp * 64; p0 < vol; p0 += 2 * nthr) {
                    int p = p0 + 2 * lane;
                    u32 two = p < vol ? *(const u32*)(bins16 + p) : 0xffffffffu;
                    int bl = p < vol ? (int)(two & 0xffffu) : -1;
                    int bh = p + 1 < vol ? (int)(two >> 16) : -1;
                    unsigned peers = __match_any_sync(0xffffffffu, bl);
                    unsigned both = __match_any_sync(0xffffffffu, bh);
                    if (bl >= 0 && lane == __ffs(peers) - 1) hist_add(hwin, A.hist, wlo, bl, (u32)__popc(peers));
                    if (bh >= 0 && lane == __ffs(both) - 1) hist_add(hwin, A.hist, wlo, bh, (u32)__popc(both));
                }
            }
            for (int wb = warp; wb < Pn.nblk; wb += nthr >> 5) {
                if (s_kind[wb] != 1 || s_nz[wb] == 0) continue;
                long long b = b0 + wb;
                int bz = (wb == Pn.nblk - 1) ? Pn.bz_last : g.e;
                int vol = rows * bz;
                const u16* bins16 = bins_all + (size_t)wb * nv8;
                TileWalk w0;
                w0.bx = Pn.bx; w0.by = Pn.by; w0.bz = bz; w0.stride = A.tile_stride; w0.zoff = wb * g.e;
                u32* unp = A.unp_scratch + (size_t)b * g.vmax;
                u32 cnt = 0;
                for (int p0 = 0; p0 < vol; p0 += 32) {
                    int p = p0 + lane;
                    bool z = p < vol && bins16[p] == 0;
                    unsigned zm = __ballot_sync(0xffffffffu, z);
                    if (z) {
                        TileWalk w = w0;
                        w.set(p);
                        unp[cnt + __popc(zm & ((1u << lane) - 1u))] = __float_as_uint(tile[w.addr()]);
                    }
                    cnt += __popc(zm);
                }
            }
        }
        __syncthreads();
        buf ^= 1;
    }
    cp_wait0();
    __syncthreads();
    hist_flush(hwin, A.hist, wlo, A.cap);
}

}  // namespace ftlz
