// blocks.cu -- per-block helpers of pipeline.compress on B200 (sm_100a) and
//   k_quant_lor stage (c) for Lorenzo blocks: one warp per block, plane wavefront (K2, Lorenzo)
// (k_prep: prep_block.cu; k_quant_reg: quant_block.cu)
// Every float64 operation is an explicit __dadd_rn/__dmul_rn (reference operand order).

namespace ftlz {

FTLZ_DEV void cp_async4(void* smem, const void* gmem) {
    unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(sa), "l"(gmem));
}
FTLZ_DEV void cp_async8(void* smem, const void* gmem) {
    unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(sa), "l"(gmem));
}
FTLZ_DEV void cp_async16(void* smem, const void* gmem) {
    unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
    asm volatile("cp.async.ca.shared.global [%0], [%1], 16;" ::"r"(sa), "l"(gmem));
}
FTLZ_DEV void cp_async_wait() { asm volatile("cp.async.wait_all;" ::: "memory"); }

FTLZ_DEV void cp_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
FTLZ_DEV void cp_wait1() { asm volatile("cp.async.wait_group 1;" ::: "memory"); }
FTLZ_DEV void cp_wait0() { asm volatile("cp.async.wait_group 0;" ::: "memory"); }

// element p (row-major in block) -> tile address, incremental walker
struct TileWalk {
    int i, j, k, bx, by, bz, stride, zoff;
    int bye;  // tile rows per i (== by for compact tiles, == box y-extent for TMA tiles)
    FTLZ_DEV void set(int p) {
        int byz = by * bz;
        i = p / byz;
        int rem = p - i * byz;
        j = rem / bz;
        k = rem - j * bz;
    }
    FTLZ_DEV int addr() const { return (i * bye + j) * stride + zoff + k; }
    FTLZ_DEV void advance(int d) {  // p += d
        k += d;
        while (k >= bz) {
            k -= bz;
            if (++j >= by) { j = 0; i++; }
        }
    }
};

// warp-cooperative single-word correction (checksum.py:109-142) over a block held in the
// tile (element p at TileWalk address); 0 clean, 1 corrected, 2 uncorrectable
FTLZ_DEV void tile_checksum(const float* tile, TileWalk w0, int vol, int lane, u64* s, u64* si) {
    u64 a = 0, c = 0;
    TileWalk w = w0;
    w.set(lane);
    for (int p = lane; p < vol; p += 32) {
        u64 v = __float_as_uint(tile[w.addr()]);
        a += v;
        c += (u64)p * v;
        w.advance(32);
    }
    *s = warp_sum_u64(a);
    *si = warp_sum_u64(c);
}

FTLZ_DEV int tile_correct(float* tile, TileWalk w0, int vol, u64 st_s, u64 st_si, int lane) {
    u64 s, si;
    tile_checksum(tile, w0, vol, lane, &s, &si);
    if (s == st_s && si == st_si) return 0;
    u64 ds = s - st_s, dsi = si - st_si;
    if (ds == 0) return 2;
    for (int j0 = 0; j0 < vol; j0 += 32) {
        int jj = j0 + lane;
        bool cand = jj < vol && (u64)jj * ds == dsi;
        unsigned m = __ballot_sync(0xffffffffu, cand);
        while (m) {
            int l = __ffs(m) - 1;
            m &= m - 1;
            TileWalk w = w0;
            w.set(j0 + l);
            int ad = w.addr();
            u64 old = __float_as_uint(tile[ad]);
            u64 restored = old - ds;
            if (restored >> 32) continue;
            __syncwarp();
            if (lane == 0) tile[ad] = __uint_as_float((u32)restored);
            __syncwarp();
            u64 s2, si2;
            tile_checksum(tile, w0, vol, lane, &s2, &si2);
            if (s2 == st_s && si2 == st_si) return 1;
            __syncwarp();
            if (lane == 0) tile[ad] = __uint_as_float((u32)old);
            __syncwarp();
        }
    }
    return 2;
}

// apply the block's INPUT faults to its tile region (one lane); returns true if any
FTLZ_DEV bool apply_input_faults(const CompArgs& A, long long b, float* tile, TileWalk w0, int lane) {
    if (!A.n_faults) return false;
    int f0 = A.fault_first[b];
    if (f0 < 0) return false;
    bool any = false;
    for (int f = f0; f < A.n_faults && A.faults[f].block == b; f++) {
        if (A.faults[f].target != FTLZ_FAULT_INPUT) continue;
        any = true;
        if (lane == 0) {
            TileWalk w = w0;
            w.set((int)A.faults[f].element);
            int ad = w.addr();
            tile[ad] = __uint_as_float(__float_as_uint(tile[ad]) ^ (1u << A.faults[f].bit));
        }
    }
    __syncwarp();
    return any;
}

// ==========================================================================================
// emit pass (both predictors), warp = block, row-major order: unpredictable words, bins
// checksum, warp-aggregated histogram, bins to the encoder layout
// CTA-window histogram increment (window of HW bins from wlo), global beyond it
template <int HW>
FTLZ_DEV void hist_add_w(u32* hwin, u64* ghist, int wlo, int bin, u32 cnt) {
    const unsigned o = (unsigned)(bin - wlo);
    if (o < (unsigned)HW) atomicAdd(&hwin[o], cnt);
    else atomicAdd(&ghist[bin], (u64)cnt);
}

template <int HW = HWIN>
FTLZ_DEV void emit_block(const CompArgs& A, long long b, int vol, const u16* bins16, const float* tile,
                         TileWalk w0, u64 dcsum, int lane, u32* hwin, int wlo) {
    const Geom& g = A.g;
    u64 bs = 0, bis = 0;
    u32 nunp = 0;
    u32* unp = A.unp_scratch + (size_t)b * g.vmax;
    size_t bidx0 = bins_index(g, b, 0);
    TileWalk w = w0;
    w.set(lane);
    for (int p0 = 0; p0 < vol; p0 += 32) {
        int p = p0 + lane;
        bool act = p < vol;
        int bin = act ? bins16[p] : -1;
        unsigned zm = __ballot_sync(0xffffffffu, bin == 0);
        if (bin == 0) unp[nunp + __popc(zm & ((1u << lane) - 1u))] = __float_as_uint(tile[w.addr()]);
        nunp += __popc(zm);
        if (act) {
            bs += (u64)bin;
            bis += (u64)p * (u64)bin;
            // [group][chunk][lane][8]: chunk p/8 advances 256 elements per 8 points
            A.bins[bidx0 + (size_t)p] = (u16)bin;
        }
        unsigned peers = __match_any_sync(0xffffffffu, bin);
        if (act && lane == __ffs(peers) - 1) hist_add_w<HW>(hwin, A.hist, wlo, bin, (u32)__popc(peers));
        w.advance(32);
    }
    dcsum = warp_sum_u64(dcsum);
    bs = warp_sum_u64(bs);
    bis = warp_sum_u64(bis);
    if (lane == 0) {
        A.unpc[b] = nunp;
        if (nunp) atomicAdd((u64*)&A.layout[LAYOUT_NUNP], (u64)nunp);
        A.bsum[b] = bs;
        A.bisum[b] = bis;
        A.dcs[b] = dcsum;
    }
}

// STAGE_DUP_EVAL fault masks of one point (ftlz_fault FTLZ_FAULT_DUP_*): XORed into the float64
// value evaluation round r returns (p = prediction, r = reconstruction)
struct DupMask {
    u64 p[3], r[3];
};

// does block b carry duplicated-evaluation faults?
FTLZ_DEV bool block_has_dup(const CompArgs& A, long long b) {
    if (!A.n_faults) return false;
    const int f0 = A.fault_first[b];
    if (f0 < 0) return false;
    for (int f = f0; f < A.n_faults && A.faults[f].block == b; f++)
        if (A.faults[f].target == FTLZ_FAULT_DUP_PREDICT || A.faults[f].target == FTLZ_FAULT_DUP_RECON) return true;
    return false;
}

// masks of point p of block b (bit = 64 * (round - 1) + b); true if any
FTLZ_DEV bool dup_masks(const CompArgs& A, long long b, int p, DupMask& m) {
    bool any = false;
#pragma unroll
    for (int r = 0; r < 3; r++) m.p[r] = m.r[r] = 0ull;
    const int f0 = A.fault_first[b];
    for (int f = f0; f >= 0 && f < A.n_faults && A.faults[f].block == b; f++) {
        const ftlz_fault F = A.faults[f];
        if (F.element != p || (F.target != FTLZ_FAULT_DUP_PREDICT && F.target != FTLZ_FAULT_DUP_RECON)) continue;
        const u64 bit = 1ull << (F.bit & 63);
        if (F.target == FTLZ_FAULT_DUP_PREDICT) m.p[F.bit >> 6] ^= bit;
        else m.r[F.bit >> 6] ^= bit;
        any = true;
    }
    return any;
}

// duplicated_eval of one element (pipeline.py:157-179): a = eval 1, b = eval 2 (dup only),
// c = eval 3 only when a != b (bitwise); the vote keeps a where a == b or a == c, else b;
// all three distinct -> *dis.  Masks model the STAGE_DUP_EVAL hook.
template <typename F2, typename F3>
FTLZ_DEV double dup_eval(double a, bool dup, F2 eval2, F3 eval3, const u64 m[3], bool* mism, bool* dis) {
    const u64 ab = dbits(a) ^ m[0];
    if (!dup) return __longlong_as_double((long long)ab);
    const u64 bb = dbits(eval2()) ^ m[1];
    if (ab == bb) return __longlong_as_double((long long)ab);
    const u64 cb = dbits(eval3()) ^ m[2];
    *mism = true;
    if (!(bb == cb || ab == cb)) *dis = true;
    return __longlong_as_double((long long)(ab == cb ? ab : bb));
}

// one point of stage (c) by the reference formulation (pipeline.py:390-409 / 416-438;
// quantize.py:37-100): pred1 / pred2 / pred3 are the three independent evaluations of the
// prediction; the reconstruction is evaluated as pred + (2 eb) * offs from independently
// loaded operands each round.  Returns the bin, writes the reconstructed value.
template <typename F2P, typename F3P>
FTLZ_DEV int quant_point(const QuantParams& Q, float x32, double p1, bool dup, F2P pred2, F3P pred3, const DupMask& M,
                         float* r32, bool* mism, double* back_out) {
    double x64 = (double)x32;
    bool pdis = false, ddis = false;
    const double pred = dup_eval(p1, dup, pred2, pred3, M.p, mism, &pdis);
    bool ok;
    int bin = quantize(Q, __dadd_rn(x64, -pred), &ok);
    if (pdis) ok = false;
    const double offs = int_to_f64(bin - Q.center);
    const double d1 = dup_eval(
        __dadd_rn(pred, __dmul_rn(Q.twoeb, offs)), dup,
        [&] { return __dadd_rn(opaque(pred), __dmul_rn(Q.twoeb_dup, opaque(offs))); },
        [&] { return __dadd_rn(opaque(opaque(pred)), __dmul_rn(opaque(Q.twoeb), opaque(opaque(offs)))); }, M.r, mism,
        &ddis);
    if (ddis) ok = false;
    float d32 = __double2float_rn(d1);
    double back = (double)d32;
    bool keep = ok && fabs(__dadd_rn(x64, -back)) <= Q.eb;
    *r32 = keep ? d32 : x32;
    *back_out = keep ? back : x64;
    return keep ? bin : 0;
}

// ==========================================================================================
// K2 (Lorenzo blocks): warp = block from the Lorenzo list; constant-(i+j+k) wavefront over a
// float64 buffer of reconstructed values (pipeline.py:199-213, 410-438)
// stage (c) of one Lorenzo block by a warp (pipeline.py:246-256,199-213): the block staged in xf
// (cp.async), input faults / stage (a) verification, the plane wavefront with the float64
// reconstruction buffer xd, the duplicated evaluation, then emit_block.  bins16 may be shared or
// global memory.  HW: the caller's CTA histogram window.
template <int HW>
FTLZ_DEV void lor_block(const CompArgs& A, const QuantParams& Q, long long b, bool dup, float* xf, double* xd,
                        u16* bins16, u32* hwin, int wlo, int lane) {
    const Geom& g = A.g;
    if (A.events[b] & 4) return;
    BlockInfo B = block_info(g, b);
    int vol = B.vol, bz = B.bz, byz = B.by * B.bz;
    // stage the block (rows of bz floats) with cp.async
    long long base = ((B.bi * g.e) * g.ny + B.bj * g.e) * g.nz + B.bk * g.e;
    {
        TileWalk w;
        w.bx = B.bx; w.by = B.by; w.bz = bz; w.stride = 0; w.zoff = 0; w.bye = B.by;
        w.set(lane);
        for (int p = lane; p < vol; p += 32) {
            cp_async4(xf + p, A.x + base + ((long long)w.i * g.ny + w.j) * g.nz + w.k);
            w.advance(32);
        }
        cp_async_wait();
    }
    __syncwarp();
    TileWalk w0;
    w0.bx = B.bx; w0.by = B.by; w0.bz = bz; w0.stride = bz * B.by; w0.zoff = 0; w0.bye = B.by;
    // block-local layout: addr = (i*by + j)*bz + k  (stride = bz per row with by rows)
    w0.stride = bz;
    if (!A.protect_input) apply_input_faults(A, b, xf, w0, lane);
    else {
        int r = tile_correct(xf, w0, vol, A.insum[b], A.inisum[b], lane);
        if (r == 1 && lane == 0) { A.events[b] |= 1; atomicAdd(&A.counters[3], 1u); }
        if (r == 2) {
            if (lane == 0) { A.events[b] |= 4; atomicAdd(&A.counters[3], 1u); }
            return;
        }
    }
    __syncwarp();
    const ExtPlan& PL = A.plans[B.xid];
    const u32* crd = A.coords + PL.coord_off;
    const u32* wave = A.wave + PL.wave_off;
    const u32* wcrd = A.wcrd + PL.wave_off;
    const u32* planes = A.planes + PL.plane_off;
    bool mism = false;
    u64 dcsum = 0;
    const bool hasdup = block_has_dup(A, b);
    const volatile double* vxd = xd;
    for (int s = 0; s < PL.nplanes; s++) {
        int q0 = __ldg(planes + s), q1 = __ldg(planes + s + 1);
        for (int q = q0 + lane; q < q1; q += 32) {
            int p = __ldg(wave + q);
            u32 c = __ldg(wcrd + q);
            int i = c & 0xff, j = (c >> 8) & 0xff, k = c >> 16;
            // the 7-term Lorenzo sum (pipeline.py:246-256); evaluations 2 and 3 re-load
            // every neighbour from the reconstruction buffer (volatile: no reuse)
            auto lor = [&](const double* buf) {
                const double d100 = i > 0 ? buf[p - byz] : 0.0;
                const double d010 = j > 0 ? buf[p - bz] : 0.0;
                const double d001 = k > 0 ? buf[p - 1] : 0.0;
                const double d110 = (i > 0 && j > 0) ? buf[p - byz - bz] : 0.0;
                const double d101 = (i > 0 && k > 0) ? buf[p - byz - 1] : 0.0;
                const double d011 = (j > 0 && k > 0) ? buf[p - bz - 1] : 0.0;
                const double d111 = (i > 0 && j > 0 && k > 0) ? buf[p - byz - bz - 1] : 0.0;
                return __dadd_rn(__dadd_rn(__dadd_rn(__dadd_rn(__dadd_rn(__dadd_rn(d100, d010), d001), -d110), -d101), -d011), d111);
            };
            auto lorv = [&]() {
                const double d100 = i > 0 ? vxd[p - byz] : 0.0;
                const double d010 = j > 0 ? vxd[p - bz] : 0.0;
                const double d001 = k > 0 ? vxd[p - 1] : 0.0;
                const double d110 = (i > 0 && j > 0) ? vxd[p - byz - bz] : 0.0;
                const double d101 = (i > 0 && k > 0) ? vxd[p - byz - 1] : 0.0;
                const double d011 = (j > 0 && k > 0) ? vxd[p - bz - 1] : 0.0;
                const double d111 = (i > 0 && j > 0 && k > 0) ? vxd[p - byz - bz - 1] : 0.0;
                return __dadd_rn(__dadd_rn(__dadd_rn(__dadd_rn(__dadd_rn(__dadd_rn(d100, d010), d001), -d110), -d101), -d011), d111);
            };
            DupMask M;
            if (hasdup) dup_masks(A, b, p, M);
            else {
#pragma unroll
                for (int r = 0; r < 3; r++) M.p[r] = M.r[r] = 0ull;
            }
            float r32;
            double back;
            int bin = quant_point(Q, xf[p], lor(xd), dup, lorv, lorv, M, &r32, &mism, &back);
            xd[p] = back;
            bins16[p] = (u16)bin;
            dcsum += __float_as_uint(r32);
        }
        __syncwarp();
    }
    if (__ballot_sync(0xffffffffu, mism) && lane == 0) atomicOr(&A.counters[1], 1u << (B.xid * 2 + 0));
    emit_block<HW>(A, b, vol, bins16, xf, w0, dcsum, lane, hwin, wlo);
    __syncwarp();
}

__global__ void __launch_bounds__(128) k_quant_lor(CompArgs A) {
    extern __shared__ __align__(16) unsigned char smem[];
    const Geom& g = A.g;
    if (dev_failed(A.st)) return;
    int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
    unsigned char* slot = smem + (size_t)warp * A.lor_slot;
    float* xf = (float*)slot;
    double* xd = (double*)(slot + (((size_t)g.vmax * 4 + 15) & ~(size_t)15));
    u16* bins16 = (u16*)(xd + g.vmax);
    u32* hwin = (u32*)(smem + (size_t)nw * A.lor_slot);
    const int wlo = A.center - HWIN / 2;
    // after k_quant_lor2d: only the blocks it deferred (faults, failed stage (a) checksum)
    const u32 n = A.lor2d ? A.counters[9] : A.counters[4];
    const u32* list = A.lor2d ? A.defer_list : A.lor_list;
    if (n == 0) return;
    for (int t = threadIdx.x; t < HWIN; t += blockDim.x) hwin[t] = 0;
    __syncthreads();
    const QuantParams Q = *A.qp;
    bool dup = A.dup_eval != 0;
    for (long long idx = (long long)blockIdx.x * nw + warp; idx < (long long)n; idx += (long long)gridDim.x * nw) {
        long long b = list[idx];
        lor_block<HWIN>(A, Q, b, dup, xf, xd, bins16, hwin, wlo, lane);
    }
    __syncthreads();
    hist_flush(hwin, A.hist, wlo, A.cap);
}

}  // namespace ftlz
