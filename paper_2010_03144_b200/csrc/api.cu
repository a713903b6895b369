// api.cu -- host runtime behind the C ABI (include/ftlz_b200.h).
//
// Unity build: the compress and decompress kernels are included here so that launch code and
// argument structs share one translation unit.  No CPU fallback exists: every entry point
// fails with FTLZ_ERR_CUDA when no device is usable.
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <map>
#include <mutex>
#include <string>
#include <tuple>
#include <vector>

#include <cudaTypedefs.h>

#include "compress.cu"
#include "blocks.cu"
#include "quant_block.cu"
#include "prep_block.cu"
#include "quant_reg10.cu"
#include "encode.cu"
#include "rle.cu"
#include "decompress.cu"
#include "decode_warp.cu"
#include "lor2d.cu"

using namespace ftlz;

// ------------------------------------------------------------------------------------------
static thread_local std::string g_err;

static int set_err(int code, const std::string& msg) {
    g_err = msg;
    return code;
}

// optional per-kernel CUDA-event timing (bench.py); events are recorded on the launch stream
struct Profiler {
    bool on = false;
    std::vector<cudaEvent_t> pool;
    size_t used = 0;
    std::vector<std::pair<std::string, cudaEvent_t>> marks;
    std::map<std::string, std::pair<double, long long>> totals;
    void mark(const char* name, cudaStream_t s) {
        if (!on) return;
        if (used == pool.size()) {
            cudaEvent_t e;
            cudaEventCreate(&e);
            pool.push_back(e);
        }
        cudaEvent_t e = pool[used++];
        cudaEventRecord(e, s);
        marks.push_back({name, e});
    }
    void collect() {  // after a stream sync
        if (!on) return;
        for (size_t i = 0; i + 1 < marks.size(); i++) {
            if (marks[i].first.empty()) continue;
            float ms = 0;
            cudaEventElapsedTime(&ms, marks[i].second, marks[i + 1].second);
            auto& t = totals[marks[i].first];
            t.first += ms;
            t.second += 1;
        }
        marks.clear();
        used = 0;
    }
};

#define LCHK(name)                                                                               \
    do {                                                                                         \
        cudaError_t e_ = cudaGetLastError();                                                     \
        if (e_ != cudaSuccess) return set_err(FTLZ_ERR_CUDA, std::string("launch ") + name + ": " + cudaGetErrorString(e_)); \
    } while (0)

#define CK(x)                                                                                    \
    do {                                                                                         \
        cudaError_t e_ = (x);                                                                    \
        if (e_ != cudaSuccess)                                                                   \
            return set_err(FTLZ_ERR_CUDA, std::string(#x) + ": " + cudaGetErrorString(e_));    \
    } while (0)

static size_t al256(size_t x) { return (x + 255) & ~(size_t)255; }

extern "C" int ftlz_abi_version(void) { return FTLZ_ABI_VERSION; }
extern "C" const char* ftlz_last_error(void) { return g_err.c_str(); }
extern "C" void ftlz_default_config(ftlz_config* c) {
    c->protect_input = c->protect_bins = c->duplicate_eval = c->store_sum_dc = 1;
    c->block_edge = 10;
    c->codec_id = 0;
    c->bin_capacity = 65536;
    c->reserved = 0;
}

extern "C" int64_t ftlz_block_count(int64_t nx, int64_t ny, int64_t nz, int32_t e) {
    if (nx < 1 || ny < 1 || nz < 1 || e < 2 || e > 64) return -1;
    return ((nx + e - 1) / e) * ((ny + e - 1) / e) * ((nz + e - 1) / e);
}

static void info_set(ftlz_info* in, int code, int kind, int64_t off, int64_t blk, int64_t a, int64_t b) {
    in->code = code; in->kind = kind; in->offset = off; in->block = blk; in->a = a; in->b = b;
}

// header validation in the reference order (container.py:189-210)
extern "C" int ftlz_peek_header(const uint8_t* d, size_t len, ftlz_header* h, ftlz_info* info) {
    info_set(info, FTLZ_OK, 0, -1, -1, 0, 0);
    auto fail = [&](int kind, int64_t off, int64_t a) {
        info_set(info, FTLZ_ERR_CORRUPT_STREAM, kind, off, -1, a, 0);
        return FTLZ_ERR_CORRUPT_STREAM;
    };
    if (len < 55) return fail(FTLZ_K_TRUNCATED, 0, FTLZ_F_HEADER);
    uint64_t nx, ny, nz, nb;
    uint32_t edge, cap;
    double eb;
    memcpy(&nx, d + 6, 8); memcpy(&ny, d + 14, 8); memcpy(&nz, d + 22, 8);
    memcpy(&edge, d + 30, 4); memcpy(&eb, d + 35, 8); memcpy(&cap, d + 43, 4); memcpy(&nb, d + 47, 8);
    if (memcmp(d, "FTLZ", 4) != 0) return fail(FTLZ_K_BAD_MAGIC, 0, 0);
    if (d[4] != 1) return fail(FTLZ_K_BAD_VERSION, 4, d[4]);
    if (nx < 1 || ny < 1 || nz < 1) return fail(FTLZ_K_BAD_DIMS, 6, 0);
    if (edge < 2 || edge > 64) return fail(FTLZ_K_BAD_EDGE, 30, edge);
    if (d[34] > 1) return fail(FTLZ_K_BAD_MODE, 34, d[34]);
    if (!(eb > 0.0 && std::isfinite(eb))) return fail(FTLZ_K_BAD_EB, 35, 0);
    if (cap < 4 || (cap & (cap - 1))) return fail(FTLZ_K_BAD_CAPACITY, 43, cap);
    unsigned __int128 expect = 1;
    bool over = false;
    uint64_t dd[3] = {nx, ny, nz};
    for (int i = 0; i < 3; i++) {
        expect *= (unsigned __int128)(dd[i] / edge + (dd[i] % edge != 0));
        if (expect >> 64) over = true;
    }
    if (over || (uint64_t)expect != nb) return fail(FTLZ_K_BLOCK_COUNT, 47, (int64_t)nb);
    h->version = d[4];
    h->codec_id = d[5];
    h->nx = (int64_t)nx; h->ny = (int64_t)ny; h->nz = (int64_t)nz;
    h->block_edge = (int32_t)edge;
    h->eb_mode = d[34];
    h->eb_value = eb;
    h->bin_capacity = cap;
    h->reserved = 0;
    h->block_count = (int64_t)nb;
    return FTLZ_OK;
}

// whole archive in host memory: header checks plus the record-table bound.  An archive too short
// for the record table its dims imply (every record takes >= 9 bytes) is truncated inside the
// table; the records are walked as container.py:212-218 reads them, so the error and its offset
// are the reference's, and no buffer is ever sized by the claimed dims of such an archive.
extern "C" int ftlz_peek_archive(const uint8_t* d, size_t len, ftlz_header* h, ftlz_info* info) {
    int rc = ftlz_peek_header(d, len, h, info);
    if (rc) return rc;
    const uint64_t nb = (uint64_t)h->block_count;
    if ((len - 55) / 9 >= nb) return FTLZ_OK;
    auto fail = [&](int kind, size_t off, int64_t a) {
        info_set(info, FTLZ_ERR_CORRUPT_STREAM, kind, (int64_t)off, -1, a, 0);
        return FTLZ_ERR_CORRUPT_STREAM;
    };
    size_t pos = 55;
    for (uint64_t b = 0; b < nb; b++) {
        if (pos + 1 > len) return fail(FTLZ_K_TRUNCATED, pos, FTLZ_F_INDICATOR);
        const uint8_t ib = d[pos];
        if (ib > 1) return fail(FTLZ_K_BAD_INDICATOR, pos, ib);
        pos += 1;
        if (ib) {
            if (pos + 16 > len) return fail(FTLZ_K_TRUNCATED, pos, FTLZ_F_COEFFS);
            pos += 16;
        }
        if (pos + 8 > len) return fail(FTLZ_K_TRUNCATED, pos, FTLZ_F_RECORD);
        pos += 8;
    }
    return FTLZ_OK;   // unreachable: the table cannot fit
}

// ------------------------------------------------------------------------------------------
// per-geometry plans: pairwise-sum leaves, coordinates, wavefront order (host built)
struct HostPlan {
    Geom g;
    ExtPlan ep[8];
    std::vector<Leaf> leaves;
    std::vector<uint32_t> coords, wave, planes;
    std::vector<uint32_t> wcrd;   // coordinates in wavefront order (same offsets as wave)
    size_t bytes() const {
        return al256(sizeof(ep)) + al256(leaves.size() * sizeof(Leaf) + 16) + al256(coords.size() * 4 + 16) +
               al256(wcrd.size() * 4 + 16) +
               al256(wave.size() * 4 + 16) + al256(planes.size() * 4 + 16);
    }
};

static void pw_leaves(int start, int n, std::vector<Leaf>& L) {
    // numpy pairwise_sum split (PW_BLOCKSIZE 128): leaves in order, combine after right subtree
    if (n <= 128) {
        L.push_back(Leaf{start, n, 0, 0});
        return;
    }
    int n2 = n / 2;
    n2 -= n2 % 8;
    pw_leaves(start, n2, L);
    pw_leaves(start + n2, n - n2, L);
    L.back().ncomb += 1;
}

static bool build_plan(int64_t nx, int64_t ny, int64_t nz, int e, HostPlan& P) {
    if (nx < 1 || ny < 1 || nz < 1 || e < 2 || e > 64) return false;
    Geom& g = P.g;
    g.nx = nx; g.ny = ny; g.nz = nz; g.e = e;
    g.cx = (nx + e - 1) / e; g.cy = (ny + e - 1) / e; g.cz = (nz + e - 1) / e;
    g.nb = g.cx * g.cy * g.cz;
    g.rx = (int)(nx - (g.cx - 1) * e); g.ry = (int)(ny - (g.cy - 1) * e); g.rz = (int)(nz - (g.cz - 1) * e);
    int mx = (int)std::min<int64_t>(e, nx), my = (int)std::min<int64_t>(e, ny), mz = (int)std::min<int64_t>(e, nz);
    g.vmax = mx * my * mz;
    g.nvmax8 = (g.vmax + 7) & ~7;
    g.fcz = make_fastdiv((u32)std::min<int64_t>(g.cz, 0xffffffffll));
    g.fcy = make_fastdiv((u32)std::min<int64_t>(g.cy, 0xffffffffll));
    P.leaves.clear(); P.coords.clear(); P.wave.clear(); P.planes.clear(); P.wcrd.clear();
    for (int xid = 0; xid < 8; xid++) {
        ExtPlan& E = P.ep[xid];
        memset(&E, 0, sizeof E);
        E.bx = (xid & 4) ? g.rx : e; E.by = (xid & 2) ? g.ry : e; E.bz = (xid & 1) ? g.rz : e;
        if (E.bx > mx) E.bx = mx;
        if (E.by > my) E.by = my;
        if (E.bz > mz) E.bz = mz;
        int vol = E.bx * E.by * E.bz;
        E.vol = vol;
        E.leaf_off = (int)P.leaves.size();
        if (vol >= 8) pw_leaves(0, vol, P.leaves);
        E.nleaf = (int)P.leaves.size() - E.leaf_off;
        E.ns = (vol - 1) / 8;
        E.sleaf_off = (int)P.leaves.size();
        if (E.ns >= 8) pw_leaves(0, E.ns, P.leaves);
        E.nsleaf = (int)P.leaves.size() - E.sleaf_off;
        {
            const int ext[3] = {E.bx, E.by, E.bz};
            const long long m = 2ll * (std::max(E.bx, std::max(E.by, E.bz)) - 1) * vol;
            E.exl = 0;
            while ((1ll << E.exl) < m) E.exl++;
            for (int ax = 0; ax < 3; ax++)
                E.den[ax] = (double)((long long)vol * ((long long)ext[ax] * ext[ax] - 1)) / 12.0;
        }
        E.coord_off = (int)P.coords.size();
        for (int i = 0; i < E.bx; i++)
            for (int j = 0; j < E.by; j++)
                for (int k = 0; k < E.bz; k++) P.coords.push_back((uint32_t)i | ((uint32_t)j << 8) | ((uint32_t)k << 16));
        E.nplanes = E.bx + E.by + E.bz - 2;
        E.wave_off = (int)P.wave.size();
        E.plane_off = (int)P.planes.size();
        std::vector<std::vector<uint32_t>> byplane(E.nplanes);
        int p = 0;
        for (int i = 0; i < E.bx; i++)
            for (int j = 0; j < E.by; j++)
                for (int k = 0; k < E.bz; k++, p++) byplane[i + j + k].push_back((uint32_t)p);
        uint32_t acc = 0;
        for (int s = 0; s < E.nplanes; s++) {
            P.planes.push_back(acc);
            for (uint32_t q : byplane[s]) {
                P.wave.push_back(q);
                P.wcrd.push_back(P.coords[E.coord_off + q]);
            }
            acc += (uint32_t)byplane[s].size();
        }
        P.planes.push_back(acc);
    }
    return true;
}

struct DevPlan {
    const ExtPlan* ep;
    const Leaf* leaves;
    const u32* coords;
    const u32* wave;
    const u32* planes;
    const u32* wcrd;
};

// upload plan tables into `dst` (device), returns pointers
static int upload_plan(const HostPlan& P, unsigned char* dst, DevPlan& D, cudaStream_t s, std::vector<unsigned char>& staging) {
    size_t off = 0;
    staging.assign(P.bytes(), 0);
    auto put = [&](const void* src, size_t n) {
        size_t o = off;
        memcpy(staging.data() + o, src, n);
        off += al256(n + 16);
        return o;
    };
    off = 0;
    size_t o_ep = 0;
    memcpy(staging.data(), P.ep, sizeof(P.ep));
    off = al256(sizeof(P.ep));
    size_t o_l = put(P.leaves.data(), P.leaves.size() * sizeof(Leaf));
    size_t o_c = put(P.coords.data(), P.coords.size() * 4);
    size_t o_w = put(P.wave.data(), P.wave.size() * 4);
    size_t o_p = put(P.planes.data(), P.planes.size() * 4);
    size_t o_wc = put(P.wcrd.data(), P.wcrd.size() * 4);
    CK(cudaMemcpyAsync(dst, staging.data(), off, cudaMemcpyHostToDevice, s));
    D.ep = (const ExtPlan*)(dst + o_ep);
    D.leaves = (const Leaf*)(dst + o_l);
    D.coords = (const u32*)(dst + o_c);
    D.wave = (const u32*)(dst + o_w);
    D.planes = (const u32*)(dst + o_p);
    D.wcrd = (const u32*)(dst + o_wc);
    return FTLZ_OK;
}

// ------------------------------------------------------------------------------------------
// kernel configuration (shared memory per block slot, blocks per CTA)
static size_t al16(size_t x) { return (x + 15) & ~(size_t)15; }

// warps of a k_decode CTA: `want`, fewer when the per-warp staging rows of a large block
// edge would not fit next to the decode table
static int dec_warps(int e, int want) {
    const size_t room = 200 * 1024 - ((size_t)4 << DEC_TBITS);
    return (int)std::max<size_t>(1, std::min<size_t>((size_t)want, room / (dec_stage_words(e) * 4)));
}

struct KCfg {
    size_t lor_smem, lor_slot;
    int lor_warps;
    StageCfg stage;
    int qr_warps, qr_slot, qr_tab, rmax;
    size_t qr_smem;
    int pp_warps, pp_slot, pp_nls, pp_ns;
    size_t pp_smem;
    int r10_slot, r10_warps;
    size_t r10_smem;
};

// TMA tensor map of the input field (dims nz, ny, nx innermost first) with a box of one block
// tile; returns 0 when the field cannot be described (rows not 16-byte aligned) -> cp.async path
static int make_input_map(CUtensorMap* m, const float* d_in, const Geom& g, const StageCfg& S) {
    static PFN_cuTensorMapEncodeTiled_v12000 enc = nullptr;
    static std::once_flag fl;
    std::call_once(fl, [] {
        void* fn = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            enc = (PFN_cuTensorMapEncodeTiled_v12000)fn;
    });
    static const bool no_tma = getenv("FTLZ_NO_TMA") != nullptr;   // debugging switch
    if (no_tma || !enc || (g.nz & 3) || ((uintptr_t)d_in & 15) || g.nz > (1ll << 32) || g.ny > (1ll << 32) ||
        g.nx > (1ll << 32) || S.tz > 256 || S.tye > 256 || S.tz > g.nz)
        return 0;
    cuuint64_t dims[3] = {(cuuint64_t)g.nz, (cuuint64_t)g.ny, (cuuint64_t)g.nx};
    cuuint64_t strides[2] = {(cuuint64_t)g.nz * 4, (cuuint64_t)g.nz * g.ny * 4};
    cuuint32_t box[3] = {(cuuint32_t)S.tz, (cuuint32_t)S.tye, (cuuint32_t)(S.box_bytes / (4 * S.tz * S.tye))};
    cuuint32_t es[3] = {1, 1, 1};
    CUresult r = enc(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, (void*)d_in, dims, strides, box, es,
                     CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                     CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS ? 1 : 0;
}

static KCfg kcfg_comp(const Geom& g) {
    KCfg k;
    size_t v = (size_t)g.vmax;
    // k_quant_reg: per-warp slots (2 TMA tiles, bins, row tables, lane histogram, mbarriers)
    {
        int ez = (int)std::min<int64_t>(g.e, g.nz);
        int maxshift = (g.e % 4 == 0) ? 0 : 4 - ((g.e % 2 == 0) ? 2 : 1);   // (bk*e) mod 4 <= this
        int tz = (ez + maxshift + 3) & ~3;
        int tye = (int)std::min<int64_t>(g.e, g.ny), txe = (int)std::min<int64_t>(g.e, g.nx);
        k.stage.use_tma = 0;
        k.stage.tz = tz;
        k.stage.tye = tye;
        k.stage.box_bytes = tz * tye * txe * 4;
        k.stage.tile_bytes = (int)((k.stage.box_bytes + 127) & ~127);
        k.stage.pad = 0;
        k.rmax = txe * tye;
        k.qr_tab = (int)al16(2 * k.stage.tile_bytes + al16(2 * (size_t)g.nvmax8));
        size_t slot = (size_t)k.qr_tab + 8 * (2 * (size_t)k.rmax + 128) + sizeof(LHT) * 32 * (LH_BINS + 1) + 16;
        slot = (slot + 127) & ~(size_t)127;
        k.qr_slot = (int)slot;
        size_t avail = 227 * 1024 - 4 * HWIN_REG - 128;
        k.qr_warps = (int)std::max<size_t>(1, std::min<size_t>(QR_WARPS, avail / slot));
        k.qr_smem = slot * k.qr_warps + 4 * HWIN_REG + 128;   // + alignment slack
        // k_prep: 2 tiles, centred-coordinate tables, fold stack, leaf partials, samples
        k.pp_nls = (int)(v / 64 + 8);
        k.pp_ns = (int)(v / 8 + 8);
        size_t ps = PREP_NBUF * (size_t)k.stage.tile_bytes +
                    8 * (6 * (size_t)g.e + 4 * PREP_STK + 4 * (size_t)k.pp_nls + 2 * (size_t)k.pp_ns) + 16;
        ps = (ps + 127) & ~(size_t)127;
        k.pp_slot = (int)ps;
        k.pp_warps = (int)std::max<size_t>(1, std::min<size_t>(20, (227 * 1024 - 256) / ps));
        k.pp_smem = ps * k.pp_warps + 128;
    }
    // k_quant_reg10: 2 TMA tiles, lane histogram (R10_LH + sink rows of 32 u8), mbarriers
    k.r10_slot = (int)(((size_t)2 * k.stage.tile_bytes + R10_LHBYTES + sizeof(R10Row) * R10_ROWS +
                        2 * sizeof(R10Pre) + 16 + 127) & ~(size_t)127);
    k.r10_warps = (int)std::max<size_t>(1, std::min<size_t>(R10_WARPS, (227 * 1024 - 4 * HWIN_REG - 256) / k.r10_slot));
    k.r10_smem = (size_t)k.r10_slot * k.r10_warps + 4 * HWIN_REG + 128;
    k.lor_slot = al16(4 * v) + 8 * v + al16(2 * v);
    k.lor_warps = (int)std::max<size_t>(1, std::min<size_t>(4, (200 * 1024) / k.lor_slot));
    k.lor_smem = k.lor_slot * k.lor_warps + 4 * HWIN;
    return k;
}

static int kernel_attrs_once() {
    static std::once_flag fl;
    static int rc = FTLZ_OK;
    std::call_once(fl, [] {
        int dev = 0;
        if (cudaGetDevice(&dev) != cudaSuccess) { rc = FTLZ_ERR_CUDA; return; }
        int maxs = 0;
        cudaDeviceGetAttribute(&maxs, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
        auto setmax = [&](const void* fn) {
            cudaFuncAttributes fa;
            if (cudaFuncGetAttributes(&fa, fn) != cudaSuccess) { rc = FTLZ_ERR_CUDA; return; }
            if (cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     maxs - (int)fa.sharedSizeBytes) != cudaSuccess)
                rc = FTLZ_ERR_CUDA;
        };
        setmax((const void*)k_prep);
        setmax((const void*)k_quant_reg);
        setmax((const void*)k_quant_reg10<false, false>);
        setmax((const void*)k_quant_reg10<false, true>);
        setmax((const void*)k_quant_reg10<true, false>);
        setmax((const void*)k_quant_reg10<true, true>);
        setmax((const void*)k_quant_lor);
        setmax((const void*)k_codebook);
        setmax((const void*)k_enc_len);
        setmax((const void*)k_enc_pack);
        setmax((const void*)k_parse_tail);
        setmax((const void*)k_decode<false, false>);
        setmax((const void*)k_decode<false, true>);
        setmax((const void*)k_recon_g<32>);
        setmax((const void*)k_recon_g<128>);
        setmax((const void*)k_redecode);
        setmax((const void*)k_decode_warp);
        setmax((const void*)k_fault_bins);
        if (cudaGetLastError() != cudaSuccess) rc = FTLZ_ERR_CUDA;
    });
    return rc;
}

static int num_sms() {
    static int n = 0;
    if (!n) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
        if (n <= 0) n = 148;
    }
    return n;
}

// ------------------------------------------------------------------------------------------
// compress workspace layout
struct CompLayout {
    size_t result;       // DevStatus | minmax[4] | counters[16] | layout[16]  (zeroed)
    size_t zero_end;
    size_t hist, lbflag, events, fixed;
    size_t coef, insum, inisum, ind, unpc, bsum, bisum, dcs, bitlen, lanepre, bitoff, regpre, unppre;
    size_t enc, qp, lbbits, lbreg, lbunp;
    size_t cb_keys, cb_syms, cb_w, cb_parent, cb_lens, cb_bm;
    size_t bins, unp, fix, faults, ffirst, ovr, plan, lor, defer, r10l, regxl;
    size_t cjobs, tarc, tarc_cap, rle, rle_bound;   // codec 1
    size_t total;
};

static const size_t RESULT_BYTES = 512;

static size_t identity_bound(const HostPlan& P, int cap) {
    const Geom& g = P.g;
    const size_t N = (size_t)g.nx * (size_t)g.ny * (size_t)g.nz, nb = (size_t)g.nb;
    const size_t nsym = std::min<size_t>((size_t)cap, N + 1);
    return 55 + 25 * nb + 4 + 5 * nsym + 8 + (57 * N + 7) / 8 + 4 * N + 16 + 8 * nb + 64;
}

static CompLayout comp_layout(const HostPlan& P, int cap, int64_t n_faults, int codec) {
    const Geom& g = P.g;
    size_t nb = (size_t)g.nb, c = (size_t)cap;
    size_t ntiles = (nb + SCAN_TILE - 1) / SCAN_TILE + 1;
    CompLayout L;
    size_t o = 0;
    auto take = [&](size_t n) { size_t r = o; o = al256(o + n); return r; };
    L.result = take(RESULT_BYTES);
    L.hist = take(8 * c);
    L.lbflag = take(4 * ntiles);
    L.events = take(nb);
    L.fixed = take(nb);
    L.cjobs = take(2 * sizeof(RleJob));
    L.cb_lens = take(c);   // code lengths (0: not in the alphabet), read whole by k_enc_len
    L.zero_end = o;
    L.coef = take(16 * nb);
    L.insum = take(8 * nb);
    L.inisum = take(8 * nb);
    L.ind = take(nb);
    L.unpc = take(4 * nb);
    L.bsum = take(8 * nb);
    L.bisum = take(8 * nb);
    L.dcs = take(8 * nb);
    L.bitlen = take(4 * nb);
    L.lanepre = take(4 * 32 * nb);
    L.bitoff = take(8 * nb);
    L.regpre = take(4 * nb);
    L.unppre = take(8 * nb);
    L.enc = take(8 * c);
    L.qp = take(sizeof(QuantParams));
    L.lbbits = take(16 * ntiles);
    L.lbreg = take(16 * ntiles);
    L.lbunp = take(16 * ntiles);
    L.cb_keys = take(16 * c);
    L.cb_syms = take(4 * c);
    L.cb_w = take(16 * c);
    L.cb_parent = take(8 * c);
    L.cb_bm = take(4 * ((c + 31) / 32));
    L.bins = take(2 * nb * (size_t)g.nvmax8 + 64);
    L.unp = take(4 * nb * (size_t)g.vmax);
    L.fix = take(n_faults ? 4 * nb * (size_t)g.vmax : 0);
    L.faults = take(sizeof(ftlz_fault) * (size_t)std::max<int64_t>(1, n_faults));
    L.ffirst = take(n_faults ? 4 * nb : 0);
    L.ovr = take(nb);
    L.lor = take(4 * nb);
    L.defer = take(4 * nb);
    L.r10l = take(4 * nb);
    L.regxl = take(4 * nb);
    L.plan = take(P.bytes());
    // codec 1: the identity archive is assembled here, then transcoded (rle.cu)
    L.tarc_cap = codec == 1 ? identity_bound(P, cap) : 0;
    L.tarc = take(L.tarc_cap);
    L.rle_bound = codec == 1 ? std::max<size_t>((57 * (size_t)g.nx * g.ny * g.nz + 7) / 8, 8 * nb) : 0;
    L.rle = take(codec == 1 ? rle_scratch_bytes(L.rle_bound) : 0);
    L.total = o;
    return L;
}

extern "C" size_t ftlz_compress_workspace_size(int64_t nx, int64_t ny, int64_t nz, const ftlz_config* cfg) {
    HostPlan P;
    if (!build_plan(nx, ny, nz, cfg->block_edge, P)) return 0;
    // faults enlarge the workspace (fix scratch); size for the faulted case
    return comp_layout(P, (int)cfg->bin_capacity, 1, cfg->codec_id).total;
}

extern "C" size_t ftlz_compress_bound(int64_t nx, int64_t ny, int64_t nz, const ftlz_config* cfg) {
    int64_t nb = ftlz_block_count(nx, ny, nz, cfg->block_edge);
    if (nb < 0) return 0;
    size_t N = (size_t)nx * ny * nz;
    size_t nsym = std::min<size_t>(cfg->bin_capacity, N + 1);
    size_t b0 = 55 + 25 * (size_t)nb + 4 + 5 * nsym + 8 + (57 * N + 7) / 8 + 4 * N + 16 + 8 * (size_t)nb + 64;
    // run-length pairs at most double the payload and the sum_dc section
    return cfg->codec_id == 1 ? b0 + (57 * N + 7) / 8 + 8 * (size_t)nb : b0;
}

// faults sorted by block + per-block first index
// faults sorted by block (stable: a block's faults keep their order)
static void prep_faults(const ftlz_fault* faults, int64_t nf, std::vector<ftlz_fault>& sorted) {
    sorted.assign(faults, faults + nf);
    std::stable_sort(sorted.begin(), sorted.end(), [](const ftlz_fault& a, const ftlz_fault& b) { return a.block < b.block; });
}

// first[b] = index of block b's first fault in the sorted list, -1 for blocks without one (the
// nb-entry table is built on the device: only the fault list crosses PCIe)
__global__ void __launch_bounds__(1024) k_fault_first(const ftlz_fault* f, int nf, long long nb, int* first) {
    // one CTA: fill, barrier, then the first fault of each block (no separate memset pass)
    for (long long b = threadIdx.x; b < nb; b += blockDim.x) first[b] = -1;
    __syncthreads();
    for (int i = threadIdx.x; i < nf; i += blockDim.x) {
        const long long b = f[i].block;
        if (b >= 0 && b < nb && (i == 0 || f[i - 1].block != b)) first[b] = i;
    }
}
// pinned staging behind a context's result buffer for the fault list and the decompressed-data
// fault blocks (a pageable H2D copy stages through the driver and costs ~10 us per call)
static size_t fault_stage_bytes(int64_t nf) { return nf ? al256(sizeof(ftlz_fault) * (size_t)nf) + al256(4 * (size_t)nf) : 0; }
// injected runs read their event flags (compress: nb bytes) or re-execution list and verdicts
// (decompress: 4 bytes per fault and the nb block flags) back with the result, into pinned room behind the staging
static size_t fault_back_bytes(int64_t nf, long long nb) { return nf ? al256((size_t)nb + 4 * (size_t)nf) : 0; }

// copy n bytes host -> device on s, through the pinned staging area when there is one (the
// stream is synchronized before the staging area is reused)
static int h2d_staged(void* dst, const void* src, size_t n, unsigned char* hstage, cudaStream_t s) {
    if (!n) return FTLZ_OK;
    if (hstage) {
        memcpy(hstage, src, n);
        src = hstage;
    }
    CK(cudaMemcpyAsync(dst, src, n, cudaMemcpyHostToDevice, s));
    return FTLZ_OK;
}

static int upload_faults(const std::vector<ftlz_fault>& fs, long long nb, unsigned char* d_faults, unsigned char* d_first,
                         cudaStream_t s, unsigned char* hstage, const void* extra = nullptr, size_t extra_n = 0) {
    const int nf = (int)fs.size();
    // extra: bytes laid out right behind the fault list on both sides (decompress: the faulted
    // block list), sent in the same copy
    const size_t fb = sizeof(ftlz_fault) * (size_t)nf;
    if (extra && extra_n && hstage) {
        memcpy(hstage, fs.data(), fb);
        memcpy(hstage + al256(fb), extra, extra_n);
        CK(cudaMemcpyAsync(d_faults, hstage, al256(fb) + extra_n, cudaMemcpyHostToDevice, s));
    } else {
        int rc = h2d_staged(d_faults, fs.data(), fb, hstage, s);
        if (rc) return rc;
        if (extra && extra_n) CK(cudaMemcpyAsync(d_faults + al256(fb), extra, extra_n, cudaMemcpyHostToDevice, s));
    }
    k_fault_first<<<1, 1024, 0, s>>>((const ftlz_fault*)d_faults, nf, nb, (int*)d_first);
    return cudaGetLastError() == cudaSuccess ? FTLZ_OK : set_err(FTLZ_ERR_CUDA, "k_fault_first");
}

static int validate_faults(const HostPlan& P, const ftlz_fault* f, int64_t nf) {
    for (int64_t i = 0; i < nf; i++) {
        if (f[i].block < 0 || f[i].block >= P.g.nb) return set_err(FTLZ_ERR_INVALID_ARGUMENT, "fault block out of range");
        int64_t b = f[i].block;
        int64_t bk = b % P.g.cz, t = b / P.g.cz, bj = t % P.g.cy, bi = t / P.g.cy;
        int xid = ((bi == P.g.cx - 1 && P.g.rx != P.g.e) ? 4 : 0) | ((bj == P.g.cy - 1 && P.g.ry != P.g.e) ? 2 : 0) |
                  ((bk == P.g.cz - 1 && P.g.rz != P.g.e) ? 1 : 0);
        int vol = P.ep[xid].vol;
        int lim = f[i].target == FTLZ_FAULT_COEFF ? 4 : f[i].target == FTLZ_FAULT_ESTIMATE ? 2 : vol;
        const bool dupf = f[i].target == FTLZ_FAULT_DUP_PREDICT || f[i].target == FTLZ_FAULT_DUP_RECON;
        int blim = f[i].target == FTLZ_FAULT_ESTIMATE ? 64 : dupf ? 192 : 32;   // dup: 64 * (round - 1) + bit
        if (f[i].element < 0 || f[i].element >= lim || f[i].bit < 0 || f[i].bit >= blim || f[i].target < 0 || f[i].target > 6)
            return set_err(FTLZ_ERR_INVALID_ARGUMENT, "fault element/bit/target out of range");
    }
    return FTLZ_OK;
}

static int block_xid(const Geom& g, int64_t b) {
    int64_t bk = b % g.cz, t = b / g.cz, bj = t % g.cy, bi = t / g.cy;
    return ((bi == g.cx - 1 && g.rx != g.e) ? 4 : 0) | ((bj == g.cy - 1 && g.ry != g.e) ? 2 : 0) |
           ((bk == g.cz - 1 && g.rz != g.e) ? 1 : 0);
}

// extent tuple for group ordering (pipeline.py:216-224)
static std::tuple<int, int, int> block_extent(const HostPlan& P, int64_t b) {
    const ExtPlan& E = P.ep[block_xid(P.g, b)];
    return std::make_tuple(E.bx, E.by, E.bz);
}

static void put_list(int64_t* dst, int64_t cap, int64_t* n_out, const std::vector<int64_t>& v) {
    *n_out = (int64_t)v.size();
    if (dst)
        for (size_t i = 0; i < v.size() && (int64_t)i < cap; i++) dst[i] = v[i];
}

static void report_reset(ftlz_report* r) {
    r->n_input_corrected = r->n_bins_corrected = r->n_dup_mismatch = r->n_reexecuted = 0;
    r->sdc = 0;
    info_set(&r->info, FTLZ_OK, 0, -1, -1, 0, 0);
    r->eb = 0; r->archive_len = 0; r->n_blocks = 0; r->n_regression = 0; r->n_unpredictable = 0;
    r->n_symbols = 0; r->payload_bits = 0; r->max_code_len = 0;
}

// ------------------------------------------------------------------------------------------
// core compress on a carved workspace.  `plan_dev` may point into the workspace (stateless
// API) or into a context cache; if `upload` the plan is copied there first.
// Optional upload overlap (UlOverlap): the host input is copied to d_in in slabs of block
// layers on a second stream, and k_prep runs on each slab as soon as it has arrived.
struct UlOverlap {
    const float* h_in = nullptr;
    cudaStream_t cs = nullptr;
    cudaEvent_t ev[8] = {};
    int nslab = 0;
};

static int compress_core(const HostPlan& P, const DevPlan* cached, const float* d_in, int32_t eb_mode,
                         double eb_value, const ftlz_config* cfg, const ftlz_fault* faults, int64_t nf,
                         const int8_t* ovr, unsigned char* ws, size_t ws_size, uint8_t* d_out, size_t out_cap,
                         ftlz_report* rep, cudaStream_t s, unsigned char* h_result, Profiler* prof = nullptr,
                         const UlOverlap* ul = nullptr) {
    Profiler noprof;
    Profiler& PF = prof ? *prof : noprof;
    report_reset(rep);
    const Geom& g = P.g;
    // context calls: h_result is pinned with fault_stage_bytes(nf) of staging behind it
    unsigned char* hstage = h_result ? h_result + RESULT_BYTES : nullptr;
    int cap = (int)cfg->bin_capacity;
    if (cap < 4 || (cap & (cap - 1))) return set_err(FTLZ_ERR_INVALID_ARGUMENT, "bin_capacity must be a power of two >= 4");
    if (cap > 65536) return set_err(FTLZ_ERR_INVALID_ARGUMENT, "bin_capacity > 65536 is not supported on the device path");
    if (cfg->codec_id != 0 && cfg->codec_id != 1) {
        info_set(&rep->info, FTLZ_ERR_UNSUPPORTED_CODEC, 0, -1, -1, cfg->codec_id, 0);
        return set_err(FTLZ_ERR_UNSUPPORTED_CODEC, "only codecs 0 (identity) and 1 (run-length) are on the device path");
    }
    int rc = validate_faults(P, faults, nf);
    if (rc) return rc;
    CompLayout L = comp_layout(P, cap, nf, cfg->codec_id);
    if (ws_size < L.total) return set_err(FTLZ_ERR_CAPACITY, "workspace too small");
    KCfg K = kcfg_comp(g);
    if (std::max(K.pp_smem, std::max(K.qr_smem, K.lor_smem)) > 227 * 1024)
        return set_err(FTLZ_ERR_INVALID_ARGUMENT, "block too large for the shared-memory path (block_edge <= 24)");
    if ((rc = kernel_attrs_once())) return set_err(rc, "cudaFuncSetAttribute failed");
    DevPlan D;
    std::vector<unsigned char> staging;
    if (cached) D = *cached;
    else if ((rc = upload_plan(P, ws + L.plan, D, s, staging))) return rc;
    CK(cudaMemsetAsync(ws, 0, L.zero_end, s));
    std::vector<ftlz_fault> fs;
    if (nf) {
        prep_faults(faults, nf, fs);
        if ((rc = upload_faults(fs, g.nb, ws + L.faults, ws + L.ffirst, s, hstage))) return rc;
    }
    if (ovr) CK(cudaMemcpyAsync(ws + L.ovr, ovr, (size_t)g.nb, cudaMemcpyHostToDevice, s));

    CompArgs A;
    memset(&A, 0, sizeof A);
    A.g = g;
    A.x = d_in;
    A.protect_input = cfg->protect_input; A.protect_bins = cfg->protect_bins;
    A.dup_eval = cfg->duplicate_eval; A.store_sum_dc = cfg->store_sum_dc;
    A.eb_mode = eb_mode; A.eb_value = eb_value;
    A.cap = cap; A.center = cap / 2;
    A.fd_e = make_fastdiv((u32)g.e); A.fd_ry = make_fastdiv((u32)g.ry);
    A.fd_rz = make_fastdiv((u32)g.rz);
    A.stage = K.stage;
    A.qr_slot = K.qr_slot;
    A.qr_tab = K.qr_tab;
    A.rmax = K.rmax;
    A.pp_slot = K.pp_slot; A.pp_nls = K.pp_nls; A.pp_ns = K.pp_ns;
    A.dbg = getenv("FTLZ_DBG") ? atoi(getenv("FTLZ_DBG")) : 0;
    CUtensorMap tmap;
    memset(&tmap, 0, sizeof tmap);
    A.stage.use_tma = make_input_map(&tmap, d_in, g, K.stage);
    // regression blocks with 10-point z rows go to k_quant_reg10 (TMA tiles of 12-float rows)
    A.r10 = (g.e == 10 && A.stage.use_tma && A.stage.tz == 12) ? 1 : 0;
    // the Lorenzo blocks ride in k_quant_reg10 when its tiles hold a block and its float64 buffer,
    // for 3-D fields of many blocks (measured on B200: c3 -61 us, c2 -62 us; the 2-D c4 and the
    // 343-block c1 are faster with k_quant_lor's own launch)
    A.lor_fused = A.r10 && g.nx > 1 && g.nb >= 4096 && A.stage.tile_bytes >= 4 * g.vmax &&
                  A.stage.tile_bytes + (int)(sizeof(R10Row) * R10_ROWS) >= 8 * g.vmax;
    // 2-D fields of 10^2 blocks: k_quant_lor2d (a lane per Lorenzo block)
    A.lor2d = !A.lor_fused && g.nx == 1 && g.e == L2_E;
    A.r10_slot = K.r10_slot;
    A.lor_slot = (int)K.lor_slot;
    A.lor_list = (u32*)(ws + L.lor);
    A.defer_list = (u32*)(ws + L.defer);
    A.r10_list = (u32*)(ws + L.r10l);
    A.regx_list = (u32*)(ws + L.regxl);
    A.n_faults = (int)nf;
    A.faults = (const ftlz_fault*)(ws + L.faults);
    A.fault_first = (const int*)(ws + L.ffirst);
    A.override_ = ovr ? (const int8_t*)(ws + L.ovr) : nullptr;
    A.plans = D.ep; A.leaves = D.leaves; A.coords = D.coords; A.wave = D.wave; A.planes = D.planes; A.wcrd = D.wcrd;
    A.coef = (float4*)(ws + L.coef); A.insum = (u64*)(ws + L.insum); A.inisum = (u64*)(ws + L.inisum);
    A.ind = ws + L.ind; A.unpc = (u32*)(ws + L.unpc); A.bsum = (u64*)(ws + L.bsum); A.bisum = (u64*)(ws + L.bisum);
    A.dcs = (u64*)(ws + L.dcs); A.bitlen = (u32*)(ws + L.bitlen); A.regpre = (u32*)(ws + L.regpre);
    A.unppre = (u64*)(ws + L.unppre); A.events = ws + L.events;
    A.lanepre = (u32*)(ws + L.lanepre); A.bitoff = (u64*)(ws + L.bitoff);
    A.st = (DevStatus*)(ws + L.result);
    A.minmax = (u32*)(ws + L.result + 64);
    A.counters = (u32*)(ws + L.result + 80);
    A.layout = (u64*)(ws + L.result + 144);
    A.qp = (QuantParams*)(ws + L.qp);
    A.hist = (u64*)(ws + L.hist);
    A.enc = (u64*)(ws + L.enc);
    A.bins = (u16*)(ws + L.bins);
    A.unp_scratch = (u32*)(ws + L.unp);
    const bool c1 = cfg->codec_id == 1;
    A.out = c1 ? ws + L.tarc : d_out;   // codec 1: identity archive in scratch, transcoded below
    A.out_cap = c1 ? L.tarc_cap : out_cap;
    CodebookScratch S;
    S.keys = (u64*)(ws + L.cb_keys); S.syms = (u32*)(ws + L.cb_syms); S.w = (u64*)(ws + L.cb_w);
    S.parent = (u32*)(ws + L.cb_parent); S.lens = ws + L.cb_lens; S.bm = (u32*)(ws + L.cb_bm);

    {
        const int nslab = ul && ul->h_in ? std::max(1, std::min<int>(ul->nslab, (int)g.cx)) : 1;
        const long long layer = g.cy * g.cz, plane = g.ny * g.nz;
        for (int si = 0; si < nslab; si++) {
            const long long l0 = g.cx * si / nslab, l1 = g.cx * (si + 1) / nslab;
            if (ul && ul->h_in) {
                const long long x0 = l0 * g.e, x1 = std::min<long long>(l1 * g.e, g.nx);
                CK(cudaMemcpyAsync((float*)d_in + x0 * plane, ul->h_in + x0 * plane, (size_t)(x1 - x0) * plane * 4,
                                   cudaMemcpyHostToDevice, ul->cs));
                CK(cudaEventRecord(ul->ev[si], ul->cs));
                CK(cudaStreamWaitEvent(s, ul->ev[si], 0));
            }
            A.pb0 = l0 * layer;
            A.pb1 = l1 * layer;
            PF.mark("k_prep", s);
            k_prep<<<(unsigned)num_sms(), 32 * K.pp_warps, K.pp_smem, s>>>(A, tmap);
            LCHK("k_prep");
        }
        A.pb0 = 0;
        A.pb1 = g.nb;
    }
    PF.mark("k_resolve", s);
    k_resolve<<<1, 1, 0, s>>>(A);
    LCHK("k_resolve");
    PF.mark("k_reglist", s);
    k_reglist<<<(unsigned)((g.nb + 1023) / 1024), 1024, 0, s>>>(A);
    LCHK("k_reglist");
    if (A.r10) {
        PF.mark("k_quant_reg10", s);
        const dim3 gr((unsigned)num_sms()), bl(32 * K.r10_warps);
        const bool dp = A.dup_eval != 0, pn = A.protect_input != 0;
        if (dp && pn) k_quant_reg10<true, true><<<gr, bl, K.r10_smem, s>>>(A, tmap);
        else if (dp) k_quant_reg10<true, false><<<gr, bl, K.r10_smem, s>>>(A, tmap);
        else if (pn) k_quant_reg10<false, true><<<gr, bl, K.r10_smem, s>>>(A, tmap);
        else k_quant_reg10<false, false><<<gr, bl, K.r10_smem, s>>>(A, tmap);
        LCHK("k_quant_reg10");
    }
    PF.mark("k_quant_reg", s);
    {
        k_quant_reg<<<(unsigned)num_sms(), 32 * K.qr_warps, K.qr_smem, s>>>(A, tmap);
    }
    LCHK("k_quant_reg");
    if (!A.lor_fused) {
        if (A.lor2d) {
            // 2-D fields: a lane per Lorenzo block; k_quant_lor then takes the deferred ones
            PF.mark("k_quant_lor2d", s);
            k_quant_lor2d<<<(unsigned)std::min<long long>((g.nb + 127) / 128, (long long)num_sms() * 16), 128, 0, s>>>(A);
            LCHK("k_quant_lor2d");
        }
        PF.mark("k_quant_lor", s);
        k_quant_lor<<<num_sms() * 4, 32 * K.lor_warps, K.lor_smem, s>>>(A);
        LCHK("k_quant_lor");
    }
    // only blocks with bins-stage faults have work in k_fault_bins
    bool bins_faults = false;
    for (const ftlz_fault& f : fs) bins_faults |= f.target == FTLZ_FAULT_BINS;
    if (bins_faults) PF.mark("k_fault_bins", s);
    if (bins_faults) {
        const int fw = (int)std::max<size_t>(1, std::min<size_t>(8, (size_t)(200 * 1024) / (4 * (size_t)g.vmax)));
        k_fault_bins<<<(unsigned)((nf + fw - 1) / fw), 32 * fw, 4 * (size_t)g.vmax * fw, s>>>(A, (u32*)(ws + L.fix),
                                                                                             (u8*)(ws + L.fixed));
    }
    LCHK("k_fault_bins");
    PF.mark("k_cb_bitmap", s);
    k_cb_bitmap<<<(unsigned)((cap + 255) / 256), 256, 0, s>>>(A, S.bm);
    PF.mark("k_codebook", s);
    k_codebook<<<1, CB_THREADS, (CB_SMEM_KEYS * 3) * 8 + CB_SMEM_KEYS * 2 * 2, s>>>(A, S);
    LCHK("k_codebook");
    {
        const size_t capal = ((size_t)cap + 15) & ~(size_t)15;
        const int lw = (int)std::max<size_t>(1, std::min<size_t>(16, (227 * 1024 / 2 - capal) / (2 * (size_t)g.nvmax8)));
        PF.mark("k_enc_len", s);
        k_enc_len<<<num_sms() * 2, 32 * lw, capal + (size_t)lw * 2 * (size_t)g.nvmax8, s>>>(
            A, (const u32*)(ws + L.fix), (const u8*)(ws + L.fixed), ws + L.cb_lens);
        LCHK("k_enc_len");
        unsigned ntiles = (unsigned)((g.nb + SCAN_TILE - 1) / SCAN_TILE);
        PF.mark("k_enc_scan", s);
        k_enc_scan<<<ntiles, SCAN_TILE, 0, s>>>(A, (u32*)(ws + L.lbflag), (u64*)(ws + L.lbbits), (u64*)(ws + L.lbreg),
                                                (u64*)(ws + L.lbunp));
        LCHK("k_enc_scan");
        PF.mark("k_enc_pack", s);
        const int pw = (int)std::max<size_t>(1, std::min<size_t>(32, (227 * 1024 - 8 * ENC_WIN - C32_BYTES) /
                                                                         (2 * (size_t)g.nvmax8 + 4 * ENC_STG)));
        k_enc_pack<<<num_sms(), 32 * pw, 8 * ENC_WIN + C32_BYTES + (size_t)pw * (2 * (size_t)g.nvmax8 + 4 * ENC_STG), s>>>(
            A, (const u32*)(ws + L.fix), (const u8*)(ws + L.fixed));
        LCHK("k_enc_pack");
    }
    ftlz_header H;
    memset(&H, 0, sizeof H);
    H.nx = g.nx; H.ny = g.ny; H.nz = g.nz; H.block_edge = g.e; H.eb_mode = eb_mode ? 1 : 0;
    PF.mark("k_assemble", s);
    k_assemble<<<num_sms() * 2, 256, 0, s>>>(A, H);
    LCHK("k_assemble");
    if (c1) {
        RleJob* jp = (RleJob*)(ws + L.cjobs);
        RleJob* js = jp + 1;
        const RleScratch RS = rle_scratch(ws + L.rle, L.rle_bound);
        PF.mark("k_rle", s);
        k_c1_prefix<<<num_sms() * 2, 256, 0, s>>>(A, d_out, out_cap, jp);
        rle_encode_launch(jp, L.rle_bound, RS, s);
        k_c1_mid<<<num_sms() * 2, 256, 0, s>>>(A, d_out, out_cap, jp, js);
        rle_encode_launch(js, L.rle_bound, RS, s);
        k_c1_fin<<<1, 1, 0, s>>>(A, d_out, out_cap, jp, js);
        LCHK("k_rle");
    }
    CK(cudaGetLastError());
    PF.mark("", s);
    unsigned char hres_local[RESULT_BYTES];
    unsigned char* hres = h_result ? h_result : hres_local;
    CK(cudaMemcpyAsync(hres, ws + L.result, RESULT_BYTES, cudaMemcpyDeviceToHost, s));
    // injected runs: the event flags come down with the result (one synchronisation)
    unsigned char* hev = nf && hstage ? hstage + fault_stage_bytes(nf) : nullptr;
    if (hev) CK(cudaMemcpyAsync(hev, ws + L.events, (size_t)g.nb, cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    PF.collect();
    DevStatus st;
    memcpy(&st, hres, sizeof st);
    u32 counters[16];
    memcpy(counters, hres + 80, sizeof counters);
    u64 lay[LAYOUT_COUNT];
    memcpy(lay, hres + 144, sizeof lay);
    double eb;
    memcpy(&eb, &lay[LAYOUT_EB_BITS], 8);
    rep->eb = eb;
    rep->n_blocks = g.nb;
    // events (rare): corrected / uncorrectable blocks
    std::vector<int64_t> in_fix, bin_fix;
    int64_t bad_in = -1, bad_bin = -1;
    if (counters[3]) {
        std::vector<unsigned char> evbuf;
        const unsigned char* ev = hev;
        if (!ev) {
            evbuf.resize((size_t)g.nb);
            CK(cudaMemcpyAsync(evbuf.data(), ws + L.events, (size_t)g.nb, cudaMemcpyDeviceToHost, s));
            CK(cudaStreamSynchronize(s));
            ev = evbuf.data();
        }
        std::tuple<int, int, int> best;
        for (int64_t b = 0; b < g.nb; b++) {
            // flags are rare: skip eight clear blocks at a time
            if (!(b & 7) && b + 8 <= g.nb) {
                u64 w8;
                memcpy(&w8, ev + b, 8);
                if (!w8) { b += 7; continue; }
            }
            if (ev[b] & 1) in_fix.push_back(b);
            if (ev[b] & 2) bin_fix.push_back(b);
            if (ev[b] & 4) {
                auto ext = block_extent(P, b);
                if (bad_in < 0 || ext < best) { bad_in = b; best = ext; }
            }
            if ((ev[b] & 8) && bad_bin < 0) bad_bin = b;
        }
    }
    if (st.code == FTLZ_ERR_DEGENERATE_BOUND) {
        info_set(&rep->info, st.code, st.kind, -1, -1, 0, 0);
        return set_err(st.code, "degenerate error bound");
    }
    if (bad_in >= 0) {
        info_set(&rep->info, FTLZ_ERR_UNCORRECTABLE, FTLZ_K_UNCORR_INPUT, -1, bad_in, 0, 0);
        return set_err(FTLZ_ERR_UNCORRECTABLE, "uncorrectable input block");
    }
    if (bad_bin >= 0) {
        info_set(&rep->info, FTLZ_ERR_UNCORRECTABLE, FTLZ_K_UNCORR_BINS_HIST, -1, bad_bin, 0, 0);
        return set_err(FTLZ_ERR_UNCORRECTABLE, "uncorrectable bin array");
    }
    if (st.code) {
        info_set(&rep->info, st.code, st.kind, st.offset, st.block, st.a, st.b);
        return set_err(st.code, "compression failed on the device");
    }
    std::vector<int64_t> dup;
    if (counters[1]) {
        std::vector<unsigned char> ind((size_t)g.nb);
        CK(cudaMemcpyAsync(ind.data(), ws + L.ind, (size_t)g.nb, cudaMemcpyDeviceToHost, s));
        CK(cudaStreamSynchronize(s));
        for (int64_t b = 0; b < g.nb; b++)
            if (counters[1] & (1u << (block_xid(g, b) * 2 + ind[b]))) dup.push_back(b);
    }
    put_list(rep->input_corrected, rep->capacity, &rep->n_input_corrected, in_fix);
    put_list(rep->bins_corrected, rep->capacity, &rep->n_bins_corrected, bin_fix);
    put_list(rep->dup_mismatch, rep->capacity, &rep->n_dup_mismatch, dup);
    rep->archive_len = (int64_t)lay[LAYOUT_TOTAL];
    rep->n_regression = (int64_t)lay[LAYOUT_NREG];
    rep->n_unpredictable = (int64_t)lay[LAYOUT_NUNP];
    rep->n_symbols = (int64_t)lay[LAYOUT_NSYM];
    rep->payload_bits = (int64_t)lay[LAYOUT_TOTAL_BITS];
    rep->max_code_len = (int32_t)lay[LAYOUT_MAXLEN];
    return FTLZ_OK;
}

extern "C" int ftlz_compress(const float* d_in, int64_t nx, int64_t ny, int64_t nz, int32_t eb_mode, double eb_value,
                             const ftlz_config* cfg, const ftlz_fault* faults, int64_t n_faults,
                             const int8_t* predictor_override, void* d_workspace, size_t workspace_size,
                             uint8_t* d_out, size_t out_capacity, ftlz_report* report, void* stream) {
    HostPlan P;
    if (!build_plan(nx, ny, nz, cfg->block_edge, P)) {
        report_reset(report);
        info_set(&report->info, FTLZ_ERR_INVALID_GEOMETRY, 0, -1, -1, 0, 0);
        return set_err(FTLZ_ERR_INVALID_GEOMETRY, "invalid dims or block edge");
    }
    return compress_core(P, nullptr, d_in, eb_mode, eb_value, cfg, faults, n_faults, predictor_override,
                         (unsigned char*)d_workspace, workspace_size, d_out, out_capacity, report,
                         (cudaStream_t)stream, nullptr);
}

// ------------------------------------------------------------------------------------------
// decompress workspace layout
struct DecLayout {
    size_t result;   // DevStatus | counters[16] | info[16]
    size_t lbflag, dflag, mflag;
    size_t zero_end;
    size_t maps, smaps, sentry;
    size_t ind, recoff, unpc, bitlen, bofs, uofs, da, db, lor, mis;
    size_t lut, lut12, lut2, first, lcount, lbase, dsym, sortkeys, lba, lbb;
    size_t bins, faults, ffirst, fblk, verdict, ckpt, plan, rlist;
    size_t jobs, payscr, sdcscr, rle;   // codec 1
    size_t pay_cap, sdc_cap, rle_bound;
    size_t total;
    long long nchunks, nsuper;
};

// codec 1 inverts the payload into a scratch of 8 bytes per point (a valid block never needs
// more than 57 bits per point) and the sum_dc section into 8 bytes per block
static DecLayout dec_layout(const HostPlan& P, size_t len, int cap, int64_t nf, int codec) {
    const Geom& g = P.g;
    size_t nb = (size_t)g.nb;
    DecLayout L;
    size_t scan = std::min<size_t>(25 * nb, len > 55 ? len - 55 : 0) + 1;
    L.nchunks = (long long)((scan + PCHUNK - 1) / PCHUNK) + 1;
    L.nsuper = (L.nchunks + PSUPER - 1) / PSUPER;
    size_t ntiles = (nb + 1023) / 1024 + 1;
    size_t o = 0;
    auto take = [&](size_t n) { size_t r = o; o = al256(o + n); return r; };
    L.result = take(RESULT_BYTES);
    L.lbflag = take(4 * ntiles);
    L.dflag = take(nb);
    L.mflag = take(nb);
    L.jobs = take(2 * sizeof(RleJob));
    L.zero_end = o;
    L.maps = take(4 * 25 * (size_t)L.nchunks);
    L.smaps = take(4 * 25 * (size_t)L.nsuper);
    L.sentry = take(8 * (size_t)L.nsuper);
    L.ind = take(nb);
    L.recoff = take(8 * nb);
    L.unpc = take(4 * nb);
    L.bitlen = take(4 * nb);
    L.bofs = take(8 * nb);
    L.uofs = take(8 * nb);
    L.da = take(8 * nb);
    L.db = take(8 * nb);
    L.lor = take(4 * nb);
    L.mis = take(4 * nb);
    L.lut = take(4 << DEC_TBITS);
    L.lut12 = take(4 << DEC_TBITS_S);
    L.lut2 = take(8 << PAIR_TBITS);
    L.first = take(8 * 64);
    L.lcount = take(4 * 64);
    L.lbase = take(4 * 64);
    L.dsym = take(4 * (size_t)cap);
    L.sortkeys = take(8 * (size_t)std::max(cap, 8192) * 2);
    L.lba = take(16 * ntiles);
    L.lbb = take(16 * ntiles);
    L.bins = take(2 * ((nb + 31) / 32) * 32 * (size_t)g.nvmax8 + 64);
    L.faults = take(sizeof(ftlz_fault) * (size_t)std::max<int64_t>(1, nf));
    L.fblk = take(4 * (size_t)std::max<int64_t>(1, nf));   // distinct faulted blocks (right behind the list: one upload)
    L.ffirst = take(nf ? 4 * nb : 0);
    L.verdict = take(nb);                                   // re-execution verdicts, list order
    L.ckpt = take(4 * RD_NCK * nb);                         // row checkpoints of the first decode
    L.plan = take(P.bytes());
    L.rlist = take(4 * nb);
    const size_t N = (size_t)g.nx * (size_t)g.ny * (size_t)g.nz;
    L.pay_cap = codec == 1 ? 8 * N + 64 : 0;
    L.sdc_cap = codec == 1 ? 8 * nb + 64 : 0;
    L.rle_bound = codec == 1 ? len : 0;
    L.payscr = take(L.pay_cap);
    L.sdcscr = take(L.sdc_cap);
    L.rle = take(codec == 1 ? rle_scratch_bytes(len) : 0);
    L.total = o;
    return L;
}

extern "C" size_t ftlz_decompress_workspace_size(const ftlz_header* h, size_t len) {
    HostPlan P;
    if (!build_plan(h->nx, h->ny, h->nz, h->block_edge, P)) return 0;
    return dec_layout(P, len, (int)std::min<uint32_t>(h->bin_capacity, 65536u), 1, h->codec_id).total;
}

struct DecResult {
    DevStatus st;
    u32 counters[16];
    u64 info[16];
};

static void stream_info_fill(const ftlz_header* h, const u64* info, ftlz_stream_info* si) {
    memset(si, 0, sizeof *si);
    si->hdr = *h;
    si->table_off = 55;
    si->table_len = (int64_t)info[DI_TABLE_END] - 55;
    si->book_off = (int64_t)info[DI_BOOK_OFF];
    si->n_symbols = (int64_t)info[DI_NSYM];
    si->payload_off = (int64_t)info[DI_PAY_OFF];
    si->payload_len = (int64_t)info[DI_PAY_LEN];
    si->unpred_off = (int64_t)info[DI_UNP_OFF];
    si->n_unpred = (int64_t)info[DI_NUNP];
    si->sumdc_off = info[DI_HAS_SDC] ? (int64_t)info[DI_SDC_OFF] : -1;
    si->total_bits = (int64_t)info[DI_TOTAL_BITS];
    si->max_code_len = (int32_t)info[DI_MAXLEN];
    si->has_sum_dc = (int32_t)info[DI_HAS_SDC];
    si->payload_stored_len = (int64_t)info[DI_PAY_STORED];
    si->sumdc_stored_len = (int64_t)info[DI_SDC_STORED];
}

// parse (+ optionally decode) on the device; d_a must have >= 64 readable bytes past len
static DecArgs make_dec_args(const HostPlan& P, const DevPlan& D, const DecLayout& L, const uint8_t* d_a, size_t len,
                             const ftlz_header* h, float* d_out, int64_t nf, unsigned char* ws) {
    const Geom& g = P.g;
    int cap = (int)h->bin_capacity;
    DecArgs A;
    memset(&A, 0, sizeof A);
    A.g = g;
    A.a = d_a;
    A.len = len;
    A.cap = cap; A.center = cap / 2;
    A.eb = h->eb_value; A.twoeb = 2.0 * h->eb_value;
    A.codec = h->codec_id;
    A.n_faults = (int)nf;
    A.faults = (const ftlz_fault*)(ws + L.faults);
    A.fault_first = (const int*)(ws + L.ffirst);
    A.ckpt = (u32*)(ws + L.ckpt);
    A.plans = D.ep; A.coords = D.coords; A.wave = D.wave; A.planes = D.planes; A.wcrd = D.wcrd;
    A.maps = (u32*)(ws + L.maps); A.smaps = (u32*)(ws + L.smaps); A.sentry = (u64*)(ws + L.sentry);
    A.nchunks = L.nchunks; A.nsuper = L.nsuper;
    A.ind = ws + L.ind; A.rec_off = (u64*)(ws + L.recoff); A.unpc = (u32*)(ws + L.unpc);
    A.bitlen = (u32*)(ws + L.bitlen); A.bofs = (u64*)(ws + L.bofs); A.uofs = (u64*)(ws + L.uofs);
    A.dflag = ws + L.dflag; A.da = (long long*)(ws + L.da); A.db = (long long*)(ws + L.db);
    A.mflag = ws + L.mflag; A.lor_list = (u32*)(ws + L.lor); A.mis_list = (u32*)(ws + L.mis);
    A.st = (DevStatus*)(ws + L.result);
    A.counters = (u32*)(ws + L.result + 64);
    A.info = (u64*)(ws + L.result + 128);
    A.lut = (u32*)(ws + L.lut); A.lut12 = (u32*)(ws + L.lut12); A.lut2 = (u64*)(ws + L.lut2); A.first_code = (u64*)(ws + L.first); A.lcount = (u32*)(ws + L.lcount);
    A.lbase = (u32*)(ws + L.lbase); A.dsym = (u32*)(ws + L.dsym); A.sortkeys = (u64*)(ws + L.sortkeys);
    A.bins = (u16*)(ws + L.bins);
    A.out = d_out;
    A.lb_flag = (u32*)(ws + L.lbflag); A.lb_a = (u64*)(ws + L.lba); A.lb_b = (u64*)(ws + L.lbb);
    A.rle_pay = (RleJob*)(ws + L.jobs); A.rle_sdc = A.rle_pay + 1;
    A.pay_scratch = ws + L.payscr; A.sdc_scratch = ws + L.sdcscr;
    A.pay_cap = L.pay_cap; A.sdc_cap = L.sdc_cap;
    A.sb0 = 0; A.sb1 = g.nb;

    return A;
}

// Optional download overlap (DlOverlap): the output is decoded in slabs of block layers and
// each finished slab is copied to h_out on a second stream while the next slab decodes.  The
// copies run before the SDC verdict is known; h_out is unspecified when the verdict withholds
// the output, and re-executed blocks are copied again afterwards.
struct DlOverlap {
    float* h_out = nullptr;
    cudaStream_t cs = nullptr;
    cudaEvent_t ev[8] = {};
    int nslab = 0;
};

// largest wavefront plane (points with i + j + k = const) of the largest block extent
static int lor_wave_max(const Geom& g) {
    const int bx = (int)std::min<int64_t>(g.e, g.nx), by = (int)std::min<int64_t>(g.e, g.ny),
              bz = (int)std::min<int64_t>(g.e, g.nz);
    int best = 0;
    for (int d = 0; d <= bx + by + bz - 3; d++) {
        int c = 0;
        for (int i = 0; i < bx; i++)
            for (int j = 0; j < by; j++) {
                const int k = d - i - j;
                c += k >= 0 && k < bz;
            }
        best = std::max(best, c);
    }
    return best;
}

static int decompress_core(const HostPlan& P, const DevPlan* cached, const uint8_t* d_a, size_t len,
                           const ftlz_header* h, float* d_out, const ftlz_fault* faults, int64_t nf,
                           unsigned char* ws, size_t ws_size, ftlz_report* rep, ftlz_stream_info* si_out,
                           bool decode, cudaStream_t s, unsigned char* h_result, Profiler* prof = nullptr,
                           const DlOverlap* dl = nullptr) {
    Profiler noprof;
    Profiler& PF = prof ? *prof : noprof;
    report_reset(rep);
    const Geom& g = P.g;
    unsigned char* hstage = h_result ? h_result + RESULT_BYTES : nullptr;   // see compress_core
    int cap = (int)h->bin_capacity;
    if (cap > 65536) return set_err(FTLZ_ERR_INVALID_ARGUMENT, "bin_capacity > 65536 is not supported on the device path");
    int rc = validate_faults(P, faults, nf);
    if (rc) return rc;
    DecLayout L = dec_layout(P, len, cap, nf, h->codec_id);
    if (ws_size < L.total) return set_err(FTLZ_ERR_CAPACITY, "workspace too small");
    if ((rc = kernel_attrs_once())) return set_err(rc, "cudaFuncSetAttribute failed");
    DevPlan D;
    std::vector<unsigned char> staging;
    if (cached) D = *cached;
    else if ((rc = upload_plan(P, ws + L.plan, D, s, staging))) return rc;
    CK(cudaMemsetAsync(ws, 0, L.zero_end, s));
    CK(cudaMemsetAsync(ws + L.result + 64 + 4 * DC_MINFAIL, 0xff, 4, s));
    std::vector<ftlz_fault> fs;
    std::vector<u32> fblk;   // distinct blocks with decompressed-data faults
    if (nf) {
        prep_faults(faults, nf, fs);
        for (const ftlz_fault& f : fs)
            if (f.target == FTLZ_FAULT_DECOMP && (fblk.empty() || fblk.back() != (u32)f.block)) fblk.push_back((u32)f.block);
        // L.fblk sits right behind L.faults: one copy
        if ((rc = upload_faults(fs, g.nb, ws + L.faults, ws + L.ffirst, s, hstage, fblk.data(), 4 * fblk.size()))) return rc;
    }
    DecArgs A = make_dec_args(P, D, L, d_a, len, h, d_out, nf, ws);
    int sms = num_sms();
    PF.mark("k_parse_chunks", s);
    k_parse_chunks<<<(unsigned)L.nsuper, 1024, 0, s>>>(A);
    LCHK("k_parse_chunks");
    PF.mark("k_parse_records", s);
    if (L.nsuper <= 256) {
        // every CTA walks the (few) super-chunk maps before its own: no k_parse_top pass
        k_parse_records<true><<<(unsigned)L.nsuper, PSUPER, 0, s>>>(A);
    } else {
        k_parse_top<<<1, 256, 0, s>>>(A);
        k_parse_records<false><<<(unsigned)L.nsuper, PSUPER, 0, s>>>(A);
    }
    LCHK("k_parse_records");
    PF.mark("k_scan2", s);
    k_scan2<<<(unsigned)((g.nb + 1023) / 1024), 1024, 0, s>>>(A);
    LCHK("k_scan2");
    PF.mark("k_parse_tail", s);
    if (h->codec_id == 1) {
        // run-length backend: invert the payload, then the sum_dc section, between the phases
        const RleScratch RS = rle_scratch(ws + L.rle, L.rle_bound);
        k_parse_tail<<<1, PT_THREADS, 8192 * 8, s>>>(A, 1);
        rle_decode_launch(A.rle_pay, L.rle_bound, RS, s);
        k_parse_tail<<<1, PT_THREADS, 8192 * 8, s>>>(A, 2);
        rle_decode_launch(A.rle_sdc, L.rle_bound, RS, s);
        k_parse_tail<<<1, PT_THREADS, 8192 * 8, s>>>(A, 3);
    } else {
        k_parse_tail<<<1, PT_THREADS, 8192 * 8, s>>>(A, 0);
    }
    LCHK("k_parse_tail");

    // full-path k_decode: up to DEC_WARPS warps per CTA, fewer when the per-warp staging rows of
    // a large block edge would not fit in shared memory
    const int dec_nw = dec_warps((int)g.e, DEC_WARPS);
    size_t dec_smem = ((size_t)4 << DEC_TBITS) + (size_t)dec_nw * dec_stage_words((int)g.e) * 4;
    int dec_occ = 0;
    CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&dec_occ, k_decode<false, true>, dec_nw * 32, dec_smem));
    dec_occ = std::max(dec_occ, 1);
    size_t rslot = al16(recon_slot_bytes(g.vmax, g.nvmax8));
    int rw = (int)std::max<size_t>(1, std::min<size_t>(4, (200 * 1024) / rslot));
    // warp-per-block decoder (decode_warp.cu) for 10^3 blocks when there are too few of them for
    // k_decode's lane per block to fill the GPU (its 1000-code chain per block is then the
    // critical path) and the archive averages at most 6 bits per point (its speculative pass
    // works per bit); k_decode otherwise, which spends fewer instructions per code.  Measured on
    // B200: c1 0.325 -> 0.037 ms, c2 0.263 -> 0.152 ms; c2 at 1e-4 (10.5 bits per point) and
    // the 2-D c4 stay on k_decode.
    const long long npts = g.nx * g.ny * g.nz;
    const bool warp_dec = decode && g.e == DW_E && g.nx >= DW_E && 2 * g.nb < (long long)num_sms() * DEC_WARPS * 32 &&
                       8 * (long long)len <= 6 * npts;
    PF.mark("k_dec_luts", s);
    k_dec_luts<<<((1u << DEC_TBITS) + (1u << DEC_TBITS_S) + (warp_dec ? 1u << PAIR_TBITS : 0u)) / 256, 256, 0, s>>>(
        A, warp_dec ? 1 : 0);
    LCHK("k_dec_luts");
    if (decode) {
        // slabs: whole block layers (block ids are layer-major), so each slab's output is one
        // contiguous range of x-planes
        // faulted runs decode in one slab: k_decomp_faults edits the output before it goes down
        const int nslab = dl && dl->h_out && fblk.empty() ? std::max(1, std::min<int>(dl->nslab, (int)g.cx)) : 1;
        const long long layer = g.cy * g.cz, plane = g.ny * g.nz;
        for (int si = 0; si < nslab; si++) {
            const long long l0 = g.cx * si / nslab, l1 = g.cx * (si + 1) / nslab;
            A.sb0 = l0 * layer;
            A.sb1 = l1 * layer;
            // one CTA per SM (fewer when there are fewer 32-block tasks), tasks split evenly
            const unsigned dgrid = (unsigned)std::min<long long>((A.sb1 - A.sb0 + 31) / 32, (long long)sms * dec_occ);
            const unsigned wgrid = (unsigned)std::min<long long>(A.sb1 - A.sb0, (long long)sms);
            PF.mark("k_decode", s);
            if (warp_dec) {
                CK(cudaMemsetAsync(ws + L.result + 64 + 4 * DC_DTICKET, 0, 4, s));
                k_decode_warp<<<wgrid, DW_WARPS * 32, DW_SMEM, s>>>(A);
            }
            else k_decode<false, true><<<dgrid, dec_nw * 32, dec_smem, s>>>(A, nullptr, 0);
            LCHK("k_decode");
            if (!fblk.empty()) {
                k_decomp_faults<<<(unsigned)((fblk.size() + 7) / 8), 256, 0, s>>>(A, (const u32*)(ws + L.fblk),
                                                                                   (int)fblk.size());
                LCHK("k_decomp_faults");
            }
            PF.mark("k_recon_warp", s);
            // a CTA per Lorenzo block when a wavefront plane exceeds a warp (10^3 blocks: up to
            // 75 points), else a warp per block (1 x e x e planes: e points) without CTA barriers
            if (g.nx == 1 && g.e == L2_E) k_recon_lor2d<<<(unsigned)std::min<long long>((g.nb + 127) / 128, (long long)sms * 16), 128, 0, s>>>(A);
            else if (lor_wave_max(g) > 32) k_recon_g<128><<<sms * 12, 128, rslot, s>>>(A, 0);
            else k_recon_g<32><<<sms * 8, rw * 32, rslot * rw, s>>>(A, 0);
            LCHK("k_recon");
            if (nslab > 1 || (dl && dl->h_out)) {
                const long long x0 = l0 * g.e, x1 = std::min<long long>(l1 * g.e, g.nx);
                CK(cudaEventRecord(dl->ev[si], s));
                CK(cudaStreamWaitEvent(dl->cs, dl->ev[si], 0));
                CK(cudaMemcpyAsync(dl->h_out + x0 * plane, d_out + x0 * plane, (size_t)(x1 - x0) * plane * 4,
                                   cudaMemcpyDeviceToHost, dl->cs));
            }
        }
        A.sb0 = 0;
        A.sb1 = g.nb;
    }
    // decompressed-data faults injected: the re-execution kernels go right behind the decode,
    // sized from the device's mismatch counter (no host round trip before them)
    const bool spec_reexec = decode && !fblk.empty();
    if (spec_reexec) {
        DecArgs AR = A;
        AR.n_faults = 0;   // re-execution replays no fault
        AR.list_spread = 0;
        PF.mark("k_reexec_decode", s);
        const size_t rsm = ((size_t)4 << DEC_TBITS_S) + (size_t)RD_WARPS * RD_MAXW * 4;
        const unsigned rg = (unsigned)std::min<size_t>((fblk.size() + RD_WARPS - 1) / RD_WARPS + 1, (size_t)sms * 4);
        k_redecode<<<rg, RD_WARPS * 32, rsm, s>>>(AR, (const u32*)(ws + L.mis), -1);
        LCHK("k_redecode");
        PF.mark("k_reexec_recon", s);
        if (lor_wave_max(g) > 32) k_recon_g<128><<<(unsigned)std::min<size_t>(fblk.size() + 1, (size_t)sms * 8), 128, rslot, s>>>(AR, 1);
        else k_recon_g<32><<<(unsigned)std::min<size_t>((fblk.size() + rw) / rw, (size_t)sms * 4), rw * 32, rslot * rw, s>>>(AR, 1);
        LCHK("k_recon");
        // context calls read the block flags back with the result and look the verdicts up on
        // the host (no verdict kernel behind the reconstruction)
        if (!hstage) {
            PF.mark("k_reexec_verdict", s);
            k_reexec_verdict<<<(unsigned)std::min<size_t>((fblk.size() + 255) / 256 + 1, 1024), 256, 0, s>>>(AR, ws + L.verdict, -1);
            LCHK("k_reexec_verdict");
        }
    }
    CK(cudaGetLastError());
    PF.mark("", s);
    unsigned char hres_local[RESULT_BYTES];
    unsigned char* hres = h_result ? h_result : hres_local;
    CK(cudaMemcpyAsync(hres, ws + L.result, RESULT_BYTES, cudaMemcpyDeviceToHost, s));
    // re-execution behind injected faults: at most one mismatching block per faulted block, so
    // the list and the verdicts come down with the result (one synchronisation)
    unsigned char* hback = spec_reexec && hstage ? hstage + fault_stage_bytes(nf) : nullptr;
    if (hback) {
        CK(cudaMemcpyAsync(hback, ws + L.mis, 4 * fblk.size(), cudaMemcpyDeviceToHost, s));
        CK(cudaMemcpyAsync(hback + 4 * fblk.size(), ws + L.mflag, (size_t)g.nb, cudaMemcpyDeviceToHost, s));
    }
    CK(cudaStreamSynchronize(s));
    PF.collect();
    DecResult R;
    memcpy(&R.st, hres, sizeof R.st);
    memcpy(R.counters, hres + 64, sizeof R.counters);
    memcpy(R.info, hres + 128, sizeof R.info);
    if (R.st.code) {
        info_set(&rep->info, R.st.code, R.st.kind, R.st.offset, R.st.block, R.st.a, R.st.b);
        return set_err(R.st.code, "archive rejected by the device parser");
    }
    if (si_out) stream_info_fill(h, R.info, si_out);
    rep->eb = h->eb_value;
    rep->n_blocks = g.nb;
    rep->n_symbols = (int64_t)R.info[DI_NSYM];
    rep->n_unpredictable = (int64_t)R.info[DI_NUNP];
    rep->payload_bits = (int64_t)R.info[DI_TOTAL_BITS];
    rep->max_code_len = (int32_t)R.info[DI_MAXLEN];
    rep->n_regression = g.nb - (int64_t)R.counters[DC_NLOR];
    rep->archive_len = (int64_t)len;
    if (!decode) return FTLZ_OK;
    if (R.counters[DC_MINFAIL] != 0xffffffffu) {
        // lowest undecodable block (pipeline.py:673-677)
        int64_t b = R.counters[DC_MINFAIL];
        unsigned char k;
        long long a2[2];
        CK(cudaMemcpyAsync(&k, ws + L.dflag + b, 1, cudaMemcpyDeviceToHost, s));
        CK(cudaStreamSynchronize(s));
        if (k == DF_PENDING) {
            // failed on the fast reader: the masked reader (which fails on exactly the same
            // blocks) names the kind and its arguments
            const u32 bb = (u32)b;
            CK(cudaMemcpyAsync(ws + L.mis, &bb, 4, cudaMemcpyHostToDevice, s));
            A.region = 1;
            A.n_faults = 0;
            k_decode<false, false><<<1, dec_nw * 32, dec_smem, s>>>(A, (const u32*)(ws + L.mis), 1);
            LCHK("k_decode");
            CK(cudaStreamSynchronize(s));
            CK(cudaMemcpyAsync(&k, ws + L.dflag + b, 1, cudaMemcpyDeviceToHost, s));
        CK(cudaStreamSynchronize(s));
            if (k == DF_PENDING) return set_err(FTLZ_ERR_INVARIANT, "fast and masked decoders disagree");
        }
        CK(cudaMemcpyAsync(&a2[0], ws + L.da + 8 * b, 8, cudaMemcpyDeviceToHost, s));
        CK(cudaStreamSynchronize(s));
        CK(cudaMemcpyAsync(&a2[1], ws + L.db + 8 * b, 8, cudaMemcpyDeviceToHost, s));
        CK(cudaStreamSynchronize(s));
        rep->sdc = 1;
        info_set(&rep->info, FTLZ_OK, k, -1, b, a2[0], a2[1]);
        return FTLZ_OK;
    }
    u32 nmis = R.counters[DC_NMIS];
    std::vector<int64_t> reexec;
    if (nmis) {
        // re-execution of every mismatching block (pipeline.py:713-723), no fault replay; the list
        // stays on the device in arrival order (blocks are independent), only the verdicts and
        // the ids come back
        A.n_faults = 0;
        if (!spec_reexec) {
        PF.mark("k_reexec_decode", s);
        {
            const size_t rsm = ((size_t)4 << DEC_TBITS_S) + (size_t)RD_WARPS * RD_MAXW * 4;
            k_redecode<<<(nmis + RD_WARPS - 1) / RD_WARPS, RD_WARPS * 32, rsm, s>>>(A, (const u32*)(ws + L.mis),
                                                                                  (int)nmis);
        }
        A.list_spread = 0;
        LCHK("k_decode");
        PF.mark("k_reexec_recon", s);
        if (lor_wave_max(g) > 32) k_recon_g<128><<<(unsigned)std::min<u32>(nmis, sms * 8), 128, rslot, s>>>(A, 1);
        else k_recon_g<32><<<(unsigned)std::min<u32>((nmis + rw - 1) / rw, sms * 4), rw * 32, rslot * rw, s>>>(A, 1);
        LCHK("k_recon");
        PF.mark("k_reexec_verdict", s);
        k_reexec_verdict<<<(nmis + 255) / 256, 256, 0, s>>>(A, ws + L.verdict, (int)nmis);
        LCHK("k_reexec_verdict");
        }
        std::vector<u32> mis(nmis);
        std::vector<unsigned char> vd(nmis);
        if (hback && nmis <= fblk.size()) {
            memcpy(mis.data(), hback, 4 * (size_t)nmis);
            const unsigned char* mf = hback + 4 * fblk.size();
            for (u32 t = 0; t < nmis; t++) vd[t] = mis[t] < (u32)g.nb ? mf[mis[t]] : 3;
        } else {
            if (hback) {   // more mismatches than faulted blocks: the verdict kernel has not run
                k_reexec_verdict<<<(nmis + 255) / 256, 256, 0, s>>>(A, ws + L.verdict, (int)nmis);
                LCHK("k_reexec_verdict");
            }
            CK(cudaMemcpyAsync(mis.data(), ws + L.mis, 4 * (size_t)nmis, cudaMemcpyDeviceToHost, s));
            CK(cudaMemcpyAsync(vd.data(), ws + L.verdict, (size_t)nmis, cudaMemcpyDeviceToHost, s));
            PF.mark("", s);
            CK(cudaStreamSynchronize(s));
            PF.collect();
        }
        // verification walks extent groups in sorted order, ids ascending (pipeline.py:692-708)
        std::vector<std::tuple<std::tuple<int, int, int>, int64_t, unsigned char>> order;
        for (u32 t = 0; t < nmis; t++) order.push_back({block_extent(P, mis[t]), (int64_t)mis[t], vd[t]});
        std::sort(order.begin(), order.end());
        for (auto& o : order) {
            const int64_t b = std::get<1>(o);
            if (std::get<2>(o) == 2) reexec.push_back(b);
            else {
                rep->sdc = 1;
                info_set(&rep->info, FTLZ_OK, FTLZ_K_D_MISMATCH, -1, b, 0, 0);
                break;
            }
        }
        std::sort(reexec.begin(), reexec.end());
        if (dl && dl->h_out && !rep->sdc) {
            // re-executed blocks changed d_out after the slab copies: copy it again
            CK(cudaStreamSynchronize(dl->cs));
            CK(cudaMemcpyAsync(dl->h_out, d_out, (size_t)g.nx * g.ny * g.nz * 4, cudaMemcpyDeviceToHost, s));
            CK(cudaStreamSynchronize(s));
        }
    }
    put_list(rep->reexecuted, rep->capacity, &rep->n_reexecuted, reexec);
    return FTLZ_OK;
}

// ------------------------------------------------------------------------------------------
// region extraction (pipeline.py:726-795), after a successful parse of the same archive in the
// same workspace: decode + reconstruct only the intersecting blocks into the region buffer,
// verify each with one re-execution, and report in the reference's processing order (extent
// groups in sorted order, block ids ascending; the first failing group stops the walk).
static int region_core(const HostPlan& P, const DevPlan& D, const uint8_t* d_a, size_t len, const ftlz_header* h,
                       const int64_t* region, float* d_out, unsigned char* ws, ftlz_report* rep, cudaStream_t s) {
    const Geom& g = P.g;
    const int cap = (int)h->bin_capacity;
    DecLayout L = dec_layout(P, len, cap, 0, h->codec_id);
    DecArgs A = make_dec_args(P, D, L, d_a, len, h, d_out, 0, ws);
    const int64_t e = g.e;
    std::vector<u32> ids;
    for (int64_t bi = region[0] / e; bi < (region[3] + e - 1) / e; bi++)
        for (int64_t bj = region[1] / e; bj < (region[4] + e - 1) / e; bj++)
            for (int64_t bk = region[2] / e; bk < (region[5] + e - 1) / e; bk++)
                ids.push_back((u32)((bi * g.cy + bj) * g.cz + bk));
    std::sort(ids.begin(), ids.end());
    const u32 n = (u32)ids.size();
    CK(cudaMemcpyAsync(ws + L.rlist, ids.data(), 4 * (size_t)n, cudaMemcpyHostToDevice, s));
    A.region = 1;
    A.rx0 = region[0]; A.ry0 = region[1]; A.rz0 = region[2];
    A.rnx = region[3] - region[0]; A.rny = region[4] - region[1]; A.rnz = region[5] - region[2];
    A.region_list = (const u32*)(ws + L.rlist);
    A.n_region = n;
    const int sms = num_sms();
    // lane per listed block, 4-warp CTAs so a short list still spreads over the SMs
    const int dnw = dec_warps((int)g.e, 4);
    const size_t dec_smem = ((size_t)4 << DEC_TBITS_S) + (size_t)dnw * dec_stage_words((int)g.e) * 4;
    const size_t rslot = al16(recon_slot_bytes(g.vmax, g.nvmax8));
    const int rw = (int)std::max<size_t>(1, std::min<size_t>(4, (200 * 1024) / rslot));
    k_decode<false, false><<<(n + dnw * 32 - 1) / (dnw * 32), dnw * 32, dec_smem, s>>>(A, A.region_list, (int)n);
    LCHK("k_decode");
    if (lor_wave_max(g) > 32) k_recon_g<128><<<std::min<u32>(n, (u32)sms * 8), 128, rslot, s>>>(A, 2);
    else k_recon_g<32><<<std::min<u32>((n + rw - 1) / rw, (u32)sms * 4), rw * 32, rslot * rw, s>>>(A, 2);
    LCHK("k_recon");
    std::vector<unsigned char> df((size_t)g.nb), mf((size_t)g.nb);
    CK(cudaMemcpyAsync(df.data(), ws + L.dflag, (size_t)g.nb, cudaMemcpyDeviceToHost, s));
    CK(cudaMemcpyAsync(mf.data(), ws + L.mflag, (size_t)g.nb, cudaMemcpyDeviceToHost, s));
    unsigned char hres[RESULT_BYTES];
    CK(cudaMemcpyAsync(hres, ws + L.result, RESULT_BYTES, cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    DevStatus st;
    memcpy(&st, hres, sizeof st);
    if (st.code) {
        info_set(&rep->info, st.code, st.kind, st.offset, st.block, st.a, st.b);
        return set_err(st.code, "device failure during region extraction");
    }
    u32 nmis = 0;
    memcpy(&nmis, hres + 64 + 4 * DC_NMIS, 4);
    if (nmis) {
        // one re-execution of every mismatching block (no fault replay)
        std::vector<u32> mis(nmis);
        CK(cudaMemcpyAsync(mis.data(), ws + L.mis, 4 * (size_t)nmis, cudaMemcpyDeviceToHost, s));
        CK(cudaStreamSynchronize(s));
        std::sort(mis.begin(), mis.end());
        CK(cudaMemcpyAsync(ws + L.mis, mis.data(), 4 * (size_t)nmis, cudaMemcpyHostToDevice, s));
        A.region = 0;   // re-decode failures mark mflag = 3
        k_decode<false, true><<<(nmis + dnw * 32 - 1) / (dnw * 32), dnw * 32, dec_smem, s>>>(
            A, (const u32*)(ws + L.mis), (int)nmis);
        LCHK("k_decode");
        if (lor_wave_max(g) > 32) k_recon_g<128><<<std::min<u32>(nmis, (u32)sms * 8), 128, rslot, s>>>(A, 3);
        else k_recon_g<32><<<std::min<u32>((nmis + rw - 1) / rw, (u32)sms * 4), rw * 32, rslot * rw, s>>>(A, 3);
        LCHK("k_recon");
        CK(cudaMemcpyAsync(mf.data(), ws + L.mflag, (size_t)g.nb, cudaMemcpyDeviceToHost, s));
        CK(cudaStreamSynchronize(s));
    }
    // verdict in processing order
    std::vector<std::pair<std::tuple<int, int, int>, int64_t>> order;
    for (u32 b : ids) order.push_back({block_extent(P, b), (int64_t)b});
    std::sort(order.begin(), order.end());
    std::vector<int64_t> reexec;
    size_t gi = 0;
    while (gi < order.size()) {
        size_t gj = gi;
        while (gj < order.size() && order[gj].first == order[gi].first) gj++;
        // undecodable blocks are raised while the group's bins are decoded, before any check
        for (size_t q = gi; q < gj; q++) {
            const int64_t b = order[q].second;
            if (df[b]) {
                long long a2[2];
                CK(cudaMemcpyAsync(&a2[0], ws + L.da + 8 * b, 8, cudaMemcpyDeviceToHost, s));
        CK(cudaStreamSynchronize(s));
                CK(cudaMemcpyAsync(&a2[1], ws + L.db + 8 * b, 8, cudaMemcpyDeviceToHost, s));
        CK(cudaStreamSynchronize(s));
                rep->sdc = 1;
                info_set(&rep->info, FTLZ_OK, df[b], -1, b, a2[0], a2[1]);
                put_list(rep->reexecuted, rep->capacity, &rep->n_reexecuted, reexec);
                return FTLZ_OK;
            }
        }
        for (size_t q = gi; q < gj; q++) {
            const int64_t b = order[q].second;
            if (mf[b] == 0) continue;
            if (mf[b] == 2) {
                reexec.push_back(b);
                continue;
            }
            rep->sdc = 1;
            info_set(&rep->info, FTLZ_OK, FTLZ_K_D_MISMATCH, -1, b, 0, 0);
            std::sort(reexec.begin(), reexec.end());
            put_list(rep->reexecuted, rep->capacity, &rep->n_reexecuted, reexec);
            return FTLZ_OK;
        }
        gi = gj;
    }
    std::sort(reexec.begin(), reexec.end());
    put_list(rep->reexecuted, rep->capacity, &rep->n_reexecuted, reexec);
    return FTLZ_OK;
}

static int region_check(const ftlz_header* h, const int64_t* r) {
    if (!(0 <= r[0] && r[0] < r[3] && r[3] <= h->nx && 0 <= r[1] && r[1] < r[4] && r[4] <= h->ny && 0 <= r[2] &&
          r[2] < r[5] && r[5] <= h->nz))
        return set_err(FTLZ_ERR_INVALID_REGION, "region outside dims");
    return FTLZ_OK;
}

extern "C" int64_t ftlz_intersecting_block_count(int64_t nx, int64_t ny, int64_t nz, int32_t block_edge,
                                                 const int64_t* r) {
    (void)nx; (void)ny; (void)nz;
    if (block_edge < 1) return -1;
    const int64_t e = block_edge;
    return ((r[3] + e - 1) / e - r[0] / e) * ((r[4] + e - 1) / e - r[1] / e) * ((r[5] + e - 1) / e - r[2] / e);
}

extern "C" int ftlz_parse(const uint8_t* d_archive, size_t len, const ftlz_header* hdr, void* d_workspace,
                          size_t workspace_size, ftlz_stream_info* info_out, ftlz_report* report, void* stream) {
    HostPlan P;
    if (!build_plan(hdr->nx, hdr->ny, hdr->nz, hdr->block_edge, P)) return set_err(FTLZ_ERR_INVALID_GEOMETRY, "bad header");
    return decompress_core(P, nullptr, d_archive, len, hdr, nullptr, nullptr, 0, (unsigned char*)d_workspace,
                           workspace_size, report, info_out, false, (cudaStream_t)stream, nullptr);
}

extern "C" int ftlz_decompress(const uint8_t* d_archive, size_t len, const ftlz_header* hdr, float* d_out,
                               const ftlz_fault* faults, int64_t n_faults, void* d_workspace, size_t workspace_size,
                               ftlz_report* report, void* stream) {
    HostPlan P;
    if (!build_plan(hdr->nx, hdr->ny, hdr->nz, hdr->block_edge, P)) return set_err(FTLZ_ERR_INVALID_GEOMETRY, "bad header");
    return decompress_core(P, nullptr, d_archive, len, hdr, d_out, faults, n_faults, (unsigned char*)d_workspace,
                           workspace_size, report, nullptr, true, (cudaStream_t)stream, nullptr);
}

// ------------------------------------------------------------------------------------------
// context API: cached device buffers, plans, pinned staging and a private stream
struct DevBuf {
    void* p = nullptr;
    size_t n = 0;
    int ensure(size_t need) {
        if (need <= n) return FTLZ_OK;
        if (p) cudaFree(p);
        p = nullptr;
        n = 0;
        size_t cap = need + need / 8 + 4096;
        cudaError_t e = cudaMalloc(&p, cap);
        if (e != cudaSuccess) return set_err(FTLZ_ERR_CUDA, std::string("cudaMalloc: ") + cudaGetErrorString(e));
        n = cap;
        return FTLZ_OK;
    }
    void release() {
        if (p) cudaFree(p);
        p = nullptr;
        n = 0;
    }
};

struct HostBuf {
    void* p = nullptr;
    size_t n = 0;
    int ensure(size_t need) {
        if (need <= n) return FTLZ_OK;
        if (p) cudaFreeHost(p);
        p = nullptr;
        n = 0;
        size_t cap = need + need / 8 + 4096;
        cudaError_t e = cudaMallocHost(&p, cap);
        if (e != cudaSuccess) return set_err(FTLZ_ERR_CUDA, std::string("cudaMallocHost: ") + cudaGetErrorString(e));
        n = cap;
        return FTLZ_OK;
    }
    void release() {
        if (p) cudaFreeHost(p);
        p = nullptr;
        n = 0;
    }
};

struct ftlz_ctx {
    int device = 0;
    cudaStream_t stream = nullptr;
    cudaStream_t cs = nullptr;   // download stream of the slab-overlapped decompress
    cudaEvent_t ev[8] = {};
    DevBuf ws, in, out, dws, arch, dout, plan, rle;
    HostBuf h_arch, h_res;
    size_t arch_len = 0;
    bool arch_on_host = false;
    // plan cache (one geometry at a time)
    int64_t pk[4] = {-1, -1, -1, -1};
    HostPlan hp;
    DevPlan dp;
    // last parsed archive (for decompress reuse)
    const uint8_t* parsed_src = nullptr;
    size_t parsed_len = 0;
    ftlz_header parsed_hdr;
    Profiler prof;
    std::mutex mu;
};

static int ctx_plan(ftlz_ctx* c, int64_t nx, int64_t ny, int64_t nz, int e) {
    if (c->pk[0] == nx && c->pk[1] == ny && c->pk[2] == nz && c->pk[3] == e) return FTLZ_OK;
    if (!build_plan(nx, ny, nz, e, c->hp)) return set_err(FTLZ_ERR_INVALID_GEOMETRY, "invalid dims or block edge");
    int rc = c->plan.ensure(c->hp.bytes());
    if (rc) return rc;
    std::vector<unsigned char> staging;
    rc = upload_plan(c->hp, (unsigned char*)c->plan.p, c->dp, c->stream, staging);
    if (rc) return rc;
    CK(cudaStreamSynchronize(c->stream));
    c->pk[0] = nx; c->pk[1] = ny; c->pk[2] = nz; c->pk[3] = e;
    return FTLZ_OK;
}

extern "C" ftlz_ctx* ftlz_ctx_create(int32_t device) {
    if (cudaSetDevice(device) != cudaSuccess) {
        set_err(FTLZ_ERR_CUDA, "cudaSetDevice failed (no usable CUDA device)");
        return nullptr;
    }
    ftlz_ctx* c = new ftlz_ctx();
    c->device = device;
    if (cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking) != cudaSuccess) {
        set_err(FTLZ_ERR_CUDA, "cudaStreamCreate failed");
        delete c;
        return nullptr;
    }
    if (c->h_res.ensure(RESULT_BYTES)) {
        delete c;
        return nullptr;
    }
    return c;
}

extern "C" void ftlz_ctx_destroy(ftlz_ctx* c) {
    if (!c) return;
    cudaSetDevice(c->device);
    cudaStreamSynchronize(c->stream);
    c->ws.release(); c->in.release(); c->out.release(); c->dws.release(); c->arch.release();
    c->dout.release(); c->plan.release(); c->rle.release(); c->h_arch.release(); c->h_res.release();
    cudaStreamDestroy(c->stream);
    if (c->cs) {
        cudaStreamSynchronize(c->cs);
        cudaStreamDestroy(c->cs);
        for (auto& e : c->ev) cudaEventDestroy(e);
    }
    delete c;
}

extern "C" void* ftlz_ctx_stream(ftlz_ctx* c) { return c ? (void*)c->stream : nullptr; }

static int ctx_compress(ftlz_ctx* c, const float* d_in, int64_t nx, int64_t ny, int64_t nz, int32_t eb_mode,
                        double eb_value, const ftlz_config* cfg, const ftlz_fault* faults, int64_t nf,
                        const int8_t* ovr, ftlz_report* rep, const UlOverlap* ul = nullptr) {
    c->prof.mark("c_host_prelude", c->stream);
    int rc = ctx_plan(c, nx, ny, nz, cfg->block_edge);
    if (rc) {
        report_reset(rep);
        info_set(&rep->info, rc, 0, -1, -1, 0, 0);
        return rc;
    }
    CompLayout L = comp_layout(c->hp, (int)cfg->bin_capacity, nf, cfg->codec_id);
    if ((rc = c->ws.ensure(L.total))) return rc;
    if ((rc = c->h_res.ensure(RESULT_BYTES + fault_stage_bytes(nf) + fault_back_bytes(nf, c->hp.g.nb)))) return rc;
    size_t bound = ftlz_compress_bound(nx, ny, nz, cfg);
    if ((rc = c->out.ensure(bound))) return rc;
    rc = compress_core(c->hp, &c->dp, d_in, eb_mode, eb_value, cfg, faults, nf, ovr, (unsigned char*)c->ws.p,
                       c->ws.n, (uint8_t*)c->out.p, c->out.n, rep, c->stream, (unsigned char*)c->h_res.p, &c->prof, ul);
    c->arch_len = rc == FTLZ_OK ? (size_t)rep->archive_len : 0;
    c->arch_on_host = false;
    return rc;
}

extern "C" int ftlz_ctx_compress_device(ftlz_ctx* c, const float* d_in, int64_t nx, int64_t ny, int64_t nz,
                                        int32_t eb_mode, double eb_value, const ftlz_config* cfg,
                                        const ftlz_fault* faults, int64_t nf, const int8_t* ovr, ftlz_report* rep) {
    std::lock_guard<std::mutex> g(c->mu);
    cudaSetDevice(c->device);
    return ctx_compress(c, d_in, nx, ny, nz, eb_mode, eb_value, cfg, faults, nf, ovr, rep);
}

// overlapped upload of a host field into c->in (UlOverlap), large fields only
static void ctx_upload_plan(ftlz_ctx* c, const float* h_in, size_t n, UlOverlap& ul) {
    if (!c->cs) {
        cudaStreamCreateWithFlags(&c->cs, cudaStreamNonBlocking);
        for (auto& e : c->ev) cudaEventCreateWithFlags(&e, cudaEventDisableTiming);
    }
    ul.h_in = h_in;
    ul.cs = c->cs;
    for (int i = 0; i < 8; i++) ul.ev[i] = c->ev[i];
    ul.nslab = n >= ((size_t)64 << 20) ? 4 : 1;
}

extern "C" int ftlz_ctx_compress_host(ftlz_ctx* c, const float* h_in, int64_t nx, int64_t ny, int64_t nz,
                                      int32_t eb_mode, double eb_value, const ftlz_config* cfg,
                                      const ftlz_fault* faults, int64_t nf, const int8_t* ovr, ftlz_report* rep) {
    std::lock_guard<std::mutex> g(c->mu);
    cudaSetDevice(c->device);
    if (nx < 1 || ny < 1 || nz < 1) {
        report_reset(rep);
        info_set(&rep->info, FTLZ_ERR_INVALID_GEOMETRY, 0, -1, -1, 0, 0);
        return set_err(FTLZ_ERR_INVALID_GEOMETRY, "invalid dims");
    }
    size_t nbytes = (size_t)nx * ny * nz * 4;
    int rc = c->in.ensure(nbytes);
    if (rc) return rc;
    UlOverlap ul;
    ctx_upload_plan(c, h_in, nbytes / 4, ul);
    rc = ctx_compress(c, (const float*)c->in.p, nx, ny, nz, eb_mode, eb_value, cfg, faults, nf, ovr, rep, &ul);
    if (rc) return rc;
    if ((rc = c->h_arch.ensure(c->arch_len))) return rc;
    CK(cudaMemcpyAsync(c->h_arch.p, c->out.p, c->arch_len, cudaMemcpyDeviceToHost, c->stream));
    CK(cudaStreamSynchronize(c->stream));
    c->arch_on_host = true;
    return FTLZ_OK;
}

extern "C" int ftlz_ctx_compress_host_to(ftlz_ctx* c, const float* h_in, int64_t nx, int64_t ny, int64_t nz,
                                         int32_t eb_mode, double eb_value, const ftlz_config* cfg,
                                         const ftlz_fault* faults, int64_t nf, const int8_t* ovr, uint8_t* h_out,
                                         size_t out_capacity, ftlz_report* rep) {
    std::lock_guard<std::mutex> g(c->mu);
    cudaSetDevice(c->device);
    if (nx < 1 || ny < 1 || nz < 1) {
        report_reset(rep);
        info_set(&rep->info, FTLZ_ERR_INVALID_GEOMETRY, 0, -1, -1, 0, 0);
        return set_err(FTLZ_ERR_INVALID_GEOMETRY, "invalid dims");
    }
    size_t nbytes = (size_t)nx * ny * nz * 4;
    int rc = c->in.ensure(nbytes);
    if (rc) return rc;
    UlOverlap ul;
    ctx_upload_plan(c, h_in, nbytes / 4, ul);
    rc = ctx_compress(c, (const float*)c->in.p, nx, ny, nz, eb_mode, eb_value, cfg, faults, nf, ovr, rep, &ul);
    if (rc) return rc;
    // the archive stays on the device for ftlz_ctx_copy_archive when it does not fit
    if (c->arch_len > out_capacity) return set_err(FTLZ_ERR_CAPACITY, "destination too small");
    CK(cudaMemcpyAsync(h_out, c->out.p, c->arch_len, cudaMemcpyDeviceToHost, c->stream));
    CK(cudaStreamSynchronize(c->stream));
    return FTLZ_OK;
}

extern "C" int ftlz_ctx_archive_device(ftlz_ctx* c, const uint8_t** d_ptr, size_t* len) {
    std::lock_guard<std::mutex> g(c->mu);
    *d_ptr = (const uint8_t*)c->out.p;
    *len = c->arch_len;
    return FTLZ_OK;
}

extern "C" int ftlz_ctx_archive_host(ftlz_ctx* c, const uint8_t** h_ptr, size_t* len) {
    std::lock_guard<std::mutex> g(c->mu);
    if (!c->arch_on_host && c->arch_len) {
        int rc = c->h_arch.ensure(c->arch_len);
        if (rc) return rc;
        CK(cudaMemcpyAsync(c->h_arch.p, c->out.p, c->arch_len, cudaMemcpyDeviceToHost, c->stream));
        CK(cudaStreamSynchronize(c->stream));
        c->arch_on_host = true;
    }
    *h_ptr = (const uint8_t*)c->h_arch.p;
    *len = c->arch_len;
    return FTLZ_OK;
}

extern "C" int ftlz_ctx_copy_archive(ftlz_ctx* c, void* h_dst, size_t capacity) {
    std::lock_guard<std::mutex> g(c->mu);
    if (capacity < c->arch_len) return set_err(FTLZ_ERR_CAPACITY, "destination too small");
    if (c->arch_on_host) {
        memcpy(h_dst, c->h_arch.p, c->arch_len);
        return FTLZ_OK;
    }
    CK(cudaMemcpyAsync(h_dst, c->out.p, c->arch_len, cudaMemcpyDeviceToHost, c->stream));
    CK(cudaStreamSynchronize(c->stream));
    return FTLZ_OK;
}

static int ctx_upload_archive(ftlz_ctx* c, const uint8_t* h, size_t len, ftlz_header* hdr, ftlz_report* rep) {
    report_reset(rep);
    c->parsed_src = nullptr;   // c->arch no longer holds the parsed archive (reuse is keyed on it)
    c->parsed_len = 0;
    int rc = ftlz_peek_archive(h, len, hdr, &rep->info);
    if (rc) return set_err(rc, "bad header");
    if ((rc = c->arch.ensure(len + 64))) return rc;
    CK(cudaMemcpyAsync(c->arch.p, h, len, cudaMemcpyHostToDevice, c->stream));
    CK(cudaMemsetAsync((unsigned char*)c->arch.p + len, 0, 64, c->stream));
    return FTLZ_OK;
}

static int ctx_decompress(ftlz_ctx* c, const uint8_t* d_a, size_t len, const ftlz_header* hdr, float* d_out,
                          const ftlz_fault* faults, int64_t nf, ftlz_report* rep, ftlz_stream_info* si, bool decode,
                          const DlOverlap* dl = nullptr) {
    c->prof.mark("d_host_prelude", c->stream);
    int rc = ctx_plan(c, hdr->nx, hdr->ny, hdr->nz, hdr->block_edge);
    if (rc) return rc;
    DecLayout L = dec_layout(c->hp, len, (int)std::min<uint32_t>(hdr->bin_capacity, 65536u), nf, hdr->codec_id);
    if ((rc = c->dws.ensure(L.total))) return rc;
    if ((rc = c->h_res.ensure(RESULT_BYTES + fault_stage_bytes(nf) + fault_back_bytes(nf, c->hp.g.nb)))) return rc;
    return decompress_core(c->hp, &c->dp, d_a, len, hdr, d_out, faults, nf, (unsigned char*)c->dws.p, c->dws.n,
                           rep, si, decode, c->stream, (unsigned char*)c->h_res.p, &c->prof, dl);
}

extern "C" int ftlz_ctx_parse_host(ftlz_ctx* c, const uint8_t* h, size_t len, ftlz_stream_info* si, ftlz_report* rep) {
    std::lock_guard<std::mutex> g(c->mu);
    cudaSetDevice(c->device);
    ftlz_header hdr;
    int rc = ctx_upload_archive(c, h, len, &hdr, rep);
    if (rc) return rc;
    rc = ctx_decompress(c, (const uint8_t*)c->arch.p, len, &hdr, nullptr, nullptr, 0, rep, si, false);
    c->parsed_src = rc == FTLZ_OK ? h : nullptr;
    c->parsed_len = len;
    c->parsed_hdr = hdr;
    return rc;
}

extern "C" int ftlz_ctx_decompress_host(ftlz_ctx* c, const uint8_t* h, size_t len, float* h_out,
                                        const ftlz_fault* faults, int64_t nf, int32_t reuse_parsed, ftlz_report* rep) {
    std::lock_guard<std::mutex> g(c->mu);
    cudaSetDevice(c->device);
    ftlz_header hdr;
    int rc;
    if (reuse_parsed && c->parsed_src == h && c->parsed_len == len) {
        hdr = c->parsed_hdr;
    } else {
        rc = ctx_upload_archive(c, h, len, &hdr, rep);
        if (rc) return rc;
    }
    size_t n = (size_t)hdr.nx * hdr.ny * hdr.nz;
    if ((rc = c->dout.ensure(4 * n))) return rc;
    // the output goes down slab by slab while later slabs decode (DlOverlap)
    if (!c->cs) {
        CK(cudaStreamCreateWithFlags(&c->cs, cudaStreamNonBlocking));
        for (auto& e : c->ev) CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    }
    DlOverlap dl;
    dl.h_out = h_out;
    dl.cs = c->cs;
    for (int i = 0; i < 8; i++) dl.ev[i] = c->ev[i];
    dl.nslab = n >= ((size_t)64 << 20) ? 4 : 1;   // small fields: one slab
    rc = ctx_decompress(c, (const uint8_t*)c->arch.p, len, &hdr, (float*)c->dout.p, faults, nf, rep, nullptr, true, &dl);
    cudaError_t ce = cudaStreamSynchronize(c->cs);
    if (rc) return rc;
    if (ce != cudaSuccess) return set_err(FTLZ_ERR_CUDA, cudaGetErrorString(ce));
    return FTLZ_OK;
}

extern "C" int ftlz_ctx_decompress_region_host(ftlz_ctx* c, const uint8_t* h, size_t len, const int64_t* region,
                                               float* h_out, int32_t reuse_parsed, ftlz_report* rep) {
    std::lock_guard<std::mutex> g(c->mu);
    cudaSetDevice(c->device);
    report_reset(rep);
    ftlz_header hdr;
    int rc;
    if (reuse_parsed && c->parsed_src == h && c->parsed_len == len) {
        hdr = c->parsed_hdr;
    } else {
        rc = ctx_upload_archive(c, h, len, &hdr, rep);
        if (rc) return rc;
    }
    if ((rc = region_check(&hdr, region))) return rc;
    // parse (validation + tables) in the context workspace, then the region pass
    rc = ctx_decompress(c, (const uint8_t*)c->arch.p, len, &hdr, nullptr, nullptr, 0, rep, nullptr, false);
    if (rc) return rc;
    const size_t n = (size_t)(region[3] - region[0]) * (region[4] - region[1]) * (region[5] - region[2]);
    if ((rc = c->dout.ensure(4 * n))) return rc;
    rc = region_core(c->hp, c->dp, (const uint8_t*)c->arch.p, len, &hdr, region, (float*)c->dout.p,
                     (unsigned char*)c->dws.p, rep, c->stream);
    if (rc) return rc;
    if (!rep->sdc) {
        CK(cudaMemcpyAsync(h_out, c->dout.p, 4 * n, cudaMemcpyDeviceToHost, c->stream));
        CK(cudaStreamSynchronize(c->stream));
    }
    return FTLZ_OK;
}

extern "C" int ftlz_ctx_decompress_device(ftlz_ctx* c, const uint8_t* d_archive, size_t len, const ftlz_header* hdr,
                                          float* d_out, const ftlz_fault* faults, int64_t nf, ftlz_report* rep) {
    std::lock_guard<std::mutex> g(c->mu);
    cudaSetDevice(c->device);
    return ctx_decompress(c, d_archive, len, hdr, d_out, faults, nf, rep, nullptr, true);
}

// ------------------------------------------------------------------------------------------
// profiling (bench.py): per-kernel event timing accumulated across calls
extern "C" int ftlz_ctx_rle_host(ftlz_ctx* c, const uint8_t* h_in, size_t n, int32_t invert, uint8_t* h_out,
                                 size_t capacity, size_t* out_len, ftlz_info* info) {
    if (!c || (!h_in && n) || !out_len) return set_err(FTLZ_ERR_INVALID_ARGUMENT, "null argument");
    std::lock_guard<std::mutex> g(c->mu);
    cudaSetDevice(c->device);
    if (info) info_set(info, FTLZ_OK, 0, -1, -1, 0, 0);
    cudaStream_t s = c->stream;
    const size_t cap = capacity;
    const size_t o_in = 0, o_out = al256(n + 64), o_job = o_out + al256(cap + 64), o_scr = o_job + 256;
    int rc = c->rle.ensure(o_scr + rle_scratch_bytes(n));
    if (rc) return rc;
    unsigned char* base = (unsigned char*)c->rle.p;
    RleJob* J = (RleJob*)(base + o_job);
    if (n) CK(cudaMemcpyAsync(base + o_in, h_in, n, cudaMemcpyHostToDevice, s));
    k_rle_setjob<<<1, 1, 0, s>>>(J, base + o_in, (u64)n, base + o_out, (u64)cap);
    const RleScratch RS = rle_scratch(base + o_scr, n);
    if (invert) rle_decode_launch(J, n, RS, s);
    else rle_encode_launch(J, n, RS, s);
    CK(cudaGetLastError());
    RleJob hj;
    CK(cudaMemcpyAsync(&hj, J, sizeof hj, cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    *out_len = (size_t)hj.out_len;
    if (invert && (hj.flags & 3u)) {
        const int k = (hj.flags & 1u) ? FTLZ_K_RLE_ODD : FTLZ_K_RLE_ZERO;
        if (info) info_set(info, FTLZ_ERR_CORRUPT_STREAM, k, -1, -1, 0, 0);
        return FTLZ_ERR_CORRUPT_STREAM;
    }
    if (hj.out_len > cap) return set_err(FTLZ_ERR_CAPACITY, "output buffer too small");
    if (hj.out_len) CK(cudaMemcpyAsync(h_out, base + o_out, (size_t)hj.out_len, cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    return FTLZ_OK;
}

extern "C" int ftlz_ctx_profile(ftlz_ctx* c, int32_t enable) {
    std::lock_guard<std::mutex> g(c->mu);
    c->prof.on = enable != 0;
    c->prof.totals.clear();
    return FTLZ_OK;
}

// writes up to max_n entries: names as '\n'-separated text, total ms and launch counts
extern "C" int ftlz_ctx_profile_read(ftlz_ctx* c, char* names, size_t names_cap, double* ms, int64_t* counts,
                                     int32_t max_n) {
    std::lock_guard<std::mutex> g(c->mu);
    std::string all;
    int n = 0;
    for (auto& kv : c->prof.totals) {
        if (n >= max_n) break;
        all += kv.first + "\n";
        ms[n] = kv.second.first;
        counts[n] = kv.second.second;
        n++;
    }
    if (all.size() + 1 > names_cap) return -1;
    memcpy(names, all.c_str(), all.size() + 1);
    return n;
}
