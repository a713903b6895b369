// rle.cu -- backend codec 1, run-length pairs (encode.py:287-312 _rle_apply / _rle_invert),
// applied by serialize to the payload and to the sum_dc section (container.py:134-145) and
// inverted by parse (container.py:241,253).
//
// Encoding: the reference scans greedily, emitting (run, byte) with run <= 255.  Equivalently,
// with s(i) the start of the maximal run of equal bytes holding position i and e(i) the start
// of the next one, position i emits a pair iff (i - s(i)) is a multiple of 255, and the pair is
// (min(255, e(i) - i), byte[i]).  The kernels tile the input (RLE_TILE bytes per CTA): tile
// bounds (first/last run start), a one-CTA pass that carries s and e across tiles, a counting
// pass, a one-CTA exclusive scan of the per-tile pair counts, and a writing pass.
// Decoding: pair k expands to run_k copies of byte_k at the exclusive prefix sum of the runs;
// an odd length or a zero run is the reference's CorruptStream, recorded in job flags.
//
// Lengths and positions are produced by earlier kernels, so every kernel reads its job from
// device memory (RleJob) and tiles past the job's length exit; grids are sized by host bounds.
namespace ftlz {

#define RLE_TPB 256
#define RLE_BPT 32
#define RLE_TILE (RLE_TPB * RLE_BPT)
#define RLE_SCAN_T 1024
#define RLE_LMAX 0x7fffffffffffffffLL

struct RleJob {
    const u8* in;
    u64 n;          // input bytes
    u8* out;
    u64 cap;        // output capacity (decode: bytes beyond it are counted, not written)
    u64 out_len;    // encoded / decoded length
    u32 flags;      // decode: 1 odd length, 2 zero-length run; encode: 4 capacity exceeded
    u32 pad;
};

// ---- CTA scans over RLE_TPB threads (8 warps)
template <typename T, typename Op>
FTLZ_DEV T cta_excl_scan(T v, T init, Op op, T* s_w, T* s_tot) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
    T inc = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const T t = __shfl_up_sync(0xffffffffu, inc, o);
        if (lane >= o) inc = op(t, inc);
    }
    if (lane == 31) s_w[warp] = inc;
    __syncthreads();
    T pre = init;
    for (int w = 0; w < warp; w++) pre = op(pre, s_w[w]);
    if (threadIdx.x == 0) {
        T tot = init;
        for (int w = 0; w < nw; w++) tot = op(tot, s_w[w]);
        *s_tot = tot;
    }
    T ex = __shfl_up_sync(0xffffffffu, inc, 1);
    ex = lane == 0 ? pre : op(pre, ex);
    __syncthreads();
    return ex;
}

// exclusive suffix scan (over threads above this one)
template <typename T, typename Op>
FTLZ_DEV T cta_excl_suffix(T v, T init, Op op, T* s_w) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
    T inc = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const T t = __shfl_down_sync(0xffffffffu, inc, o);
        if (lane + o < 32) inc = op(inc, t);
    }
    if (lane == 0) s_w[warp] = inc;
    __syncthreads();
    T suf = init;
    for (int w = nw - 1; w > warp; w--) suf = op(suf, s_w[w]);
    T ex = __shfl_down_sync(0xffffffffu, inc, 1);
    ex = lane == 31 ? suf : op(ex, suf);
    __syncthreads();
    return ex;
}

// tile bytes [a - 1, a + RLE_TILE) into shared memory with aligned 16-byte loads; returns the
// shift: byte a + k - 1 sits at s[shift + k].  The 16-byte chunks around the ends stay inside
// the buffer's allocation (device buffers are 256-byte aligned and padded past their end).
#define RLE_SBUF (RLE_TILE + 48)
FTLZ_DEV int rle_load_tile(const u8* in, u64 n, u64 a, u8* s) {
    const u8* lo = in + a - (a ? 1 : 0);
    const u8* base = (const u8*)((uintptr_t)lo & ~(uintptr_t)15);
    const u64 end = min(n, a + (u64)RLE_TILE);
    const u64 nch = ((uintptr_t)(in + end) - (uintptr_t)base + 15) >> 4;
    for (u64 c = threadIdx.x; c < nch; c += blockDim.x) ((uint4*)s)[c] = __ldg((const uint4*)base + c);
    __syncthreads();
    return (int)((uintptr_t)lo - (uintptr_t)base) - (a ? 0 : 1);
}

FTLZ_DEV bool rle_start(const u8* s, int sh, u64 a, int k) {
    return (a == 0 && k == 0) || s[sh + k + 1] != s[sh + k];
}

// per tile: first and last run start (-1: none)
__global__ void __launch_bounds__(RLE_TPB) k_rle_bounds(const RleJob* J, long long* tfirst, long long* tlast) {
    __shared__ __align__(16) u8 s[RLE_SBUF];
    __shared__ long long s_w[8], s_t;
    const u64 n = J->n;
    for (u64 t = blockIdx.x; t * RLE_TILE < n; t += gridDim.x) {
    const u64 a = t * RLE_TILE;
    const int sh = rle_load_tile(J->in, n, a, s);
    long long f = RLE_LMAX, l = -1;
    const int k0 = threadIdx.x * RLE_BPT;
    for (int k = k0; k < k0 + RLE_BPT && a + k < n; k++)
        if (rle_start(s, sh, a, k)) {
            if (f == RLE_LMAX) f = (long long)(a + k);
            l = (long long)(a + k);
        }
    auto mn = [](long long x, long long y) { return x < y ? x : y; };
    auto mx = [](long long x, long long y) { return x > y ? x : y; };
    cta_excl_scan<long long>(f, RLE_LMAX, mn, s_w, &s_t);
    const long long fmin = s_t;
    __syncthreads();
    cta_excl_scan<long long>(l, -1LL, mx, s_w, &s_t);
    if (threadIdx.x == 0) {
        tfirst[t] = fmin;
        tlast[t] = s_t;
    }
    __syncthreads();
    }
}

// one CTA: run start carried into each tile (exclusive prefix max of tile lasts) and the first
// run start after each tile (exclusive suffix min of tile firsts, n when none)
__global__ void __launch_bounds__(RLE_SCAN_T) k_rle_carry(const RleJob* J, const long long* tfirst, const long long* tlast,
                                                          long long* cs, long long* ce) {
    __shared__ long long s_w[32], s_t;
    const u64 n = J->n;
    const long long nt = (long long)((n + RLE_TILE - 1) / RLE_TILE);
    auto mn = [](long long x, long long y) { return x < y ? x : y; };
    auto mx = [](long long x, long long y) { return x > y ? x : y; };
    long long carry = -1;
    for (long long c0 = 0; c0 < nt; c0 += blockDim.x) {
        const long long t = c0 + threadIdx.x;
        const long long v = t < nt ? tlast[t] : -1;
        const long long ex = cta_excl_scan<long long>(v, carry, mx, s_w, &s_t);
        if (t < nt) cs[t] = ex;
        carry = s_t;
        __syncthreads();
    }
    long long carry2 = (long long)n;
    const long long nch = (nt + blockDim.x - 1) / blockDim.x;
    for (long long ci = nch - 1; ci >= 0; ci--) {
        const long long t = ci * blockDim.x + threadIdx.x;
        const long long v = t < nt ? tfirst[t] : RLE_LMAX;
        const long long ex = cta_excl_suffix<long long>(v, carry2, mn, s_w);
        if (t < nt) ce[t] = ex;
        // the chunk's total for the next (lower) chunk: min over its tiles and the carry
        long long m = v;
        for (int o = 16; o > 0; o >>= 1) m = mn(m, __shfl_xor_sync(0xffffffffu, m, o));
        if ((threadIdx.x & 31) == 0) s_w[threadIdx.x >> 5] = m;
        __syncthreads();
        if (threadIdx.x == 0) {
            long long r = carry2;
            for (int w = 0; w < (int)(blockDim.x >> 5); w++) r = mn(r, s_w[w]);
            s_t = r;
        }
        __syncthreads();
        carry2 = s_t;
        __syncthreads();
    }
}

// counting (WRITE = false: per-tile pair counts) and writing (WRITE = true) passes
template <bool WRITE>
__global__ void __launch_bounds__(RLE_TPB) k_rle_emit(RleJob* J, const long long* cs, const long long* ce, u64* tcount,
                                                      const u64* toff) {
    __shared__ __align__(16) u8 s[RLE_SBUF];
    __shared__ u8 st[WRITE ? 2 * RLE_TILE : 1];
    __shared__ long long s_w[8], s_t;
    __shared__ u64 s_wu[8], s_tu;
    const u64 n = J->n;
    for (u64 t = blockIdx.x; t * RLE_TILE < n; t += gridDim.x) {
    const u64 a = t * RLE_TILE;
    const int sh = rle_load_tile(J->in, n, a, s);
    const int k0 = threadIdx.x * RLE_BPT;
    const int k1 = (int)min((u64)(k0 + RLE_BPT), n - a > (u64)RLE_TILE ? (u64)RLE_TILE : n - a);
    long long f = RLE_LMAX, l = -1;
    for (int k = k0; k < k1; k++)
        if (rle_start(s, sh, a, k)) {
            if (f == RLE_LMAX) f = (long long)(a + k);
            l = (long long)(a + k);
        }
    auto mn = [](long long x, long long y) { return x < y ? x : y; };
    auto mx = [](long long x, long long y) { return x > y ? x : y; };
    const long long sb = cta_excl_scan<long long>(l, cs[t], mx, s_w, &s_t);   // run start before k0
    const long long ea = cta_excl_suffix<long long>(f, ce[t], mn, s_w);        // next start at/after k1
    // ascending: emission mask (bit k - k0)
    u32 mask = 0;
    if (k0 < k1) {
        u32 m = (u32)(((long long)(a + k0) - sb) % 255);
        for (int k = k0; k < k1; k++) {
            if (rle_start(s, sh, a, k)) m = 0;
            if (m == 0) mask |= 1u << (k - k0);
            m = m + 1 == 255 ? 0 : m + 1;
        }
    }
    const u64 cnt = (u64)__popc(mask);
    auto add = [](u64 x, u64 y) { return x + y; };
    const u64 pre = cta_excl_scan<u64>(cnt, 0ull, add, s_wu, &s_tu);
    if (!WRITE) {
        if (threadIdx.x == 0) tcount[t] = s_tu;
        __syncthreads();
        continue;
    }
    // pairs of the tile staged in shared memory (at most 2 bytes per input byte), then one
    // coalesced copy to the tile's output range
    const u64 tbase = toff[t], tpairs = s_tu;
    u8* const out = J->out;
    const bool fits = 2 * (tbase + tpairs) <= J->cap;
    if (!fits && threadIdx.x == 0 && tpairs) atomicOr(&J->flags, 4u);
    long long nxt = ea;
    for (int k = k1 - 1; k >= k0; k--) {
        const long long i = (long long)(a + k);
        const long long e = nxt;
        if (rle_start(s, sh, a, k)) nxt = i;
        if ((mask >> (k - k0)) & 1u) {
            const u64 r = pre + (u64)__popc(mask & ((1u << (k - k0)) - 1u));
            const long long run = e - i < 255 ? e - i : 255;
            st[2 * r] = (u8)run;
            st[2 * r + 1] = s[sh + k + 1];
        }
    }
    __syncthreads();
    if (fits)
        for (u64 q = threadIdx.x; q < 2 * tpairs; q += blockDim.x) out[2 * tbase + q] = st[q];
    __syncthreads();
    }
}

// one CTA: exclusive scan of per-tile counts (encode: pairs; decode: decoded bytes)
__global__ void __launch_bounds__(RLE_SCAN_T) k_rle_offsets(RleJob* J, const u64* tcount, u64* toff, int decode) {
    __shared__ u64 s_w[32], s_t;
    const u64 n = decode ? (J->n & ~1ull) : J->n;   // decode: whole pairs only (odd: error)
    const long long nt = (long long)((n + RLE_TILE - 1) / RLE_TILE);
    auto add = [](u64 x, u64 y) { return x + y; };
    u64 carry = 0;
    for (long long c0 = 0; c0 < nt; c0 += blockDim.x) {
        const long long t = c0 + threadIdx.x;
        const u64 v = t < nt ? tcount[t] : 0;
        const u64 ex = cta_excl_scan<u64>(v, carry, add, s_w, &s_t);
        if (t < nt) toff[t] = ex;
        carry = s_t;
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        if (decode) {
            J->out_len = carry;
            if (J->n & 1) J->flags |= 1u;
        } else {
            J->out_len = 2 * carry;
            if (2 * carry > J->cap) J->flags |= 4u;
        }
    }
}

// decode: per tile (RLE_TILE stored bytes = RLE_TILE / 2 pairs) the decoded byte count and
// whether a zero run occurs
__global__ void __launch_bounds__(RLE_TPB) k_rld_sums(RleJob* J, u64* tcount) {
    __shared__ u64 s_wu[8], s_tu;
    const u64 n = J->n & ~1ull;
    for (u64 t = blockIdx.x; t * RLE_TILE < n; t += gridDim.x) {
    const u64 a = t * RLE_TILE;
    u64 sum = 0;
    bool zero = false;
    for (u64 k = a + 2 * threadIdx.x; k < a + RLE_TILE && k < n; k += 2 * blockDim.x) {
        const u32 r = J->in[k];
        sum += r;
        zero |= r == 0;
    }
    auto add = [](u64 x, u64 y) { return x + y; };
    cta_excl_scan<u64>(sum, 0ull, add, s_wu, &s_tu);
    if (__syncthreads_or(zero) && threadIdx.x == 0) atomicOr(&J->flags, 2u);
    if (threadIdx.x == 0) tcount[t] = s_tu;
    __syncthreads();
    }
}

// decode: expand the pairs of each tile at their offsets (bytes past the capacity are dropped)
__global__ void __launch_bounds__(RLE_TPB) k_rld_write(RleJob* J, const u64* toff) {
    __shared__ u64 s_wu[8], s_tu;
    const u64 n = J->n & ~1ull;
    u8* const out = J->out;
    const u64 cap = J->cap;
    for (u64 t = blockIdx.x; t * RLE_TILE < n; t += gridDim.x) {
    const u64 a = t * RLE_TILE;
    const u64 k0 = a + (u64)threadIdx.x * RLE_BPT;
    u64 sum = 0;
    for (u64 k = k0; k < k0 + RLE_BPT && k < n; k += 2) sum += J->in[k];
    auto add = [](u64 x, u64 y) { return x + y; };
    u64 o = toff[t] + cta_excl_scan<u64>(sum, 0ull, add, s_wu, &s_tu);
    for (u64 k = k0; k < k0 + RLE_BPT && k < n; k += 2) {
        const u32 r = J->in[k];
        const u8 v = J->in[k + 1];
        for (u32 q = 0; q < r && o + q < cap; q++) out[o + q] = v;
        o += r;
    }
    }
}

// ---- host side: scratch layout and launch sequences (job filled on the device beforehand)
struct RleScratch {
    long long *tfirst, *tlast, *cs, *ce;
    u64 *tcount, *toff;
};

static size_t rle_tiles(size_t n_bound) { return (n_bound + RLE_TILE - 1) / RLE_TILE + 1; }
static size_t rle_scratch_bytes(size_t n_bound) { return 6 * 8 * rle_tiles(n_bound) + 256; }
static RleScratch rle_scratch(unsigned char* p, size_t n_bound) {
    const size_t t = rle_tiles(n_bound);
    RleScratch R;
    R.tfirst = (long long*)p;
    R.tlast = R.tfirst + t;
    R.cs = R.tlast + t;
    R.ce = R.cs + t;
    R.tcount = (u64*)(R.ce + t);
    R.toff = R.tcount + t;
    return R;
}

// tile kernels loop over tiles (the job's length is only known on the device)
static unsigned rle_grid(size_t n_bound) {
    static int sms = 0;
    if (!sms) {
        int d = 0;
        cudaGetDevice(&d);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, d);
        if (sms <= 0) sms = 148;
    }
    return (unsigned)std::min<size_t>(rle_tiles(n_bound), (size_t)sms * 8);
}

static void rle_encode_launch(RleJob* J, size_t n_bound, const RleScratch& R, cudaStream_t s) {
    const unsigned nt = rle_grid(n_bound);
    k_rle_bounds<<<nt, RLE_TPB, 0, s>>>(J, R.tfirst, R.tlast);
    k_rle_carry<<<1, RLE_SCAN_T, 0, s>>>(J, R.tfirst, R.tlast, R.cs, R.ce);
    k_rle_emit<false><<<nt, RLE_TPB, 0, s>>>(J, R.cs, R.ce, R.tcount, R.toff);
    k_rle_offsets<<<1, RLE_SCAN_T, 0, s>>>(J, R.tcount, R.toff, 0);
    k_rle_emit<true><<<nt, RLE_TPB, 0, s>>>(J, R.cs, R.ce, R.tcount, R.toff);
}

static void rle_decode_launch(RleJob* J, size_t n_bound, const RleScratch& R, cudaStream_t s) {
    const unsigned nt = rle_grid(n_bound);
    k_rld_sums<<<nt, RLE_TPB, 0, s>>>(J, R.tcount);
    k_rle_offsets<<<1, RLE_SCAN_T, 0, s>>>(J, R.tcount, R.toff, 1);
    k_rld_write<<<nt, RLE_TPB, 0, s>>>(J, R.toff);
}

// standalone job (host-known input): fill, run, read back
__global__ void k_rle_setjob(RleJob* J, const u8* in, u64 n, u8* out, u64 cap) {
    J->in = in;
    J->n = n;
    J->out = out;
    J->cap = cap;
    J->out_len = 0;
    J->flags = 0;
}

}  // namespace ftlz

// ---- codec 1 on the compress side: the identity archive is assembled in a scratch buffer
//      (A.out), then transcoded into the caller's buffer: prefix (header with codec byte 1,
//      block table, codebook), u64 stored length + run-length payload, unpredictable words,
//      (raw, stored) lengths + run-length sum_dc (container.py:109-147)
namespace ftlz {

__global__ void k_c1_prefix(CompArgs A, u8* dst, u64 dst_cap, RleJob* jp) {
    if (dev_failed(A.st)) return;
    const u64 n = A.layout[LAYOUT_PAYLEN_OFF], pay_off = A.layout[LAYOUT_PAY_OFF];
    if (n + 8 > dst_cap) return;   // reported by k_c1_fin
    for (u64 i = (u64)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (u64)gridDim.x * blockDim.x)
        dst[i] = i == 5 ? (u8)1 : A.out[i];
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        jp->in = A.out + pay_off;
        jp->n = A.layout[LAYOUT_PAY_BYTES];
        jp->out = dst + pay_off;
        jp->cap = dst_cap > pay_off ? dst_cap - pay_off : 0;
        jp->out_len = 0;
        jp->flags = 0;
    }
}

__global__ void k_c1_mid(CompArgs A, u8* dst, u64 dst_cap, const RleJob* jp, RleJob* js) {
    if (dev_failed(A.st) || (jp->flags & 4u)) return;
    const u64 pay_off = A.layout[LAYOUT_PAY_OFF], stored = jp->out_len;
    const u64 unp_src = A.layout[LAYOUT_UNP_OFF], nunp_b = 4 * A.layout[LAYOUT_NUNP];
    const u64 unp_dst = pay_off + stored;
    const u64 lens = unp_dst + nunp_b;
    if (lens + 16 > dst_cap) return;
    for (u64 i = (u64)blockIdx.x * blockDim.x + threadIdx.x; i < nunp_b; i += (u64)gridDim.x * blockDim.x)
        dst[unp_dst + i] = A.out[unp_src + i];
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        const u64 paylen_off = A.layout[LAYOUT_PAYLEN_OFF];
        for (int q = 0; q < 8; q++) dst[paylen_off + q] = (u8)(stored >> (8 * q));
        js->in = A.out + A.layout[LAYOUT_SDC_OFF] + 16;
        js->n = A.store_sum_dc ? 8ull * (u64)A.g.nb : 0ull;
        js->out = dst + lens + 16;
        js->cap = dst_cap - (lens + 16);
        js->out_len = 0;
        js->flags = 0;
    }
}

__global__ void k_c1_fin(CompArgs A, u8* dst, u64 dst_cap, const RleJob* jp, const RleJob* js) {
    if (dev_failed(A.st)) return;
    const u64 pay_off = A.layout[LAYOUT_PAY_OFF], stored = jp->out_len;
    const u64 lens = pay_off + stored + 4 * A.layout[LAYOUT_NUNP];
    const u64 raw = A.store_sum_dc ? 8ull * (u64)A.g.nb : 0ull, sst = raw ? js->out_len : 0ull;
    const u64 total = lens + 16 + sst;
    if ((jp->flags & 4u) || (js->flags & 4u) || A.layout[LAYOUT_PAYLEN_OFF] + 8 > dst_cap || total > dst_cap) {
        dev_fail(A.st, FTLZ_ERR_CAPACITY, 0, -1, -1, (long long)total, 0, 0);
        return;
    }
    for (int q = 0; q < 8; q++) {
        dst[lens + q] = (u8)(raw >> (8 * q));
        dst[lens + 8 + q] = (u8)(sst >> (8 * q));
    }
    A.layout[LAYOUT_TOTAL] = total;
}

}  // namespace ftlz
