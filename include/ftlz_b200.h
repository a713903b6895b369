/*
 * ftlz_b200.h -- C ABI of the B200-native FT-SZ (SDC-resilient SZ) compress/decompress path.
 *
 * The reference (`ftlz` 0.1.0, pure Python, /root/reference/pkg/src/ftlz) has no FFI; its
 * drop-in boundary is the Python API re-exported by __init__.py:6-38.  Every entry point
 * below replaces one reference function; the Python mirror in paper_2010_03144_b200/ binds
 * them with ctypes (see INTEGRATION.md for the binding a maintainer would add).
 *
 *   ftlz_compress / ftlz_ctx_compress_*   <- pipeline.compress  (pipeline.py:287-537)
 *                                            + container.serialize (container.py:109-147);
 *                                            the device emits the serialized archive directly.
 *   ftlz_peek_header                      <- container.parse header checks (container.py:176-210)
 *   ftlz_ctx_parse_*                      <- container.parse (container.py:173-285), validation
 *                                            of records / codebook / sections on the device.
 *   ftlz_decompress / ftlz_ctx_decompress_* <- pipeline.decompress (pipeline.py:645-723)
 *
 * Conventions: plain pointers and sizes only; `stream` is a cudaStream_t passed as void*.
 * Status codes map 1:1 to the reference exception classes (errors.py:4-59).  A terminal SDC in
 * decompression is NOT an error status: it is reported in ftlz_report.sdc (pipeline.py:673-677,
 * 704-707), exactly as the reference returns (None, report) instead of raising.
 * The library keeps no pointer to caller buffers after a call returns.
 */
#ifndef FTLZ_B200_H
#define FTLZ_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define FTLZ_ABI_VERSION 3

/* ---- status codes (errors.py:4-59) ------------------------------------------------------- */
enum ftlz_status {
    FTLZ_OK = 0,
    FTLZ_ERR_INVALID_GEOMETRY = 1,  /* InvalidGeometry            */
    FTLZ_ERR_DEGENERATE_BOUND = 2,  /* DegenerateBound            */
    FTLZ_ERR_UNCORRECTABLE = 3,     /* UncorrectableCorruption    */
    FTLZ_ERR_INVARIANT = 4,         /* InternalInvariantViolation */
    FTLZ_ERR_CORRUPT_STREAM = 5,    /* CorruptStream(offset)      */
    FTLZ_ERR_UNSUPPORTED_CODEC = 6, /* UnsupportedCodec           */
    FTLZ_ERR_INVALID_ARGUMENT = 7,  /* InvalidArgument            */
    FTLZ_ERR_CUDA = 8,              /* CUDA runtime failure (no reference counterpart) */
    FTLZ_ERR_CAPACITY = 9,          /* caller buffer too small    */
    FTLZ_ERR_INVALID_REGION = 10    /* InvalidRegion              */
};

/* ---- detail kinds: select the reference message text ------------------------------------ */
enum ftlz_kind {
    FTLZ_K_NONE = 0,
    /* compression */
    FTLZ_K_UNCORR_INPUT = 1,       /* "input block {block} failed verification beyond repair" (pipeline.py:343) */
    FTLZ_K_UNCORR_BINS_HIST = 2,   /* "bin array of block {block} ... (histogram)" (pipeline.py:477) */
    FTLZ_K_UNCORR_BINS_ENC = 3,    /* "... (encode)" */
    FTLZ_K_BIN_RANGE = 4,          /* "bin index outside quantizer range" (pipeline.py:490) */
    FTLZ_K_CODE_LEN = 5,           /* "code length {a} exceeds cap 57" (encode.py:85-88) */
    FTLZ_K_DEGENERATE = 6,         /* resolved bound not positive/finite (core.py:188-192); eb in report */
    /* container.parse (container.py:173-285); offset field carries the reference offset */
    FTLZ_K_TRUNCATED = 20,         /* "truncated while reading {what=a}" */
    FTLZ_K_BAD_MAGIC = 21,
    FTLZ_K_BAD_VERSION = 22,
    FTLZ_K_BAD_DIMS = 23,
    FTLZ_K_BAD_EDGE = 24,
    FTLZ_K_BAD_MODE = 25,
    FTLZ_K_BAD_EB = 26,
    FTLZ_K_BAD_CAPACITY = 27,
    FTLZ_K_BLOCK_COUNT = 28,
    FTLZ_K_BAD_INDICATOR = 29,     /* a = indicator byte */
    FTLZ_K_SYM_ORDER = 30,
    FTLZ_K_SYM_RANGE = 31,         /* a = symbol */
    FTLZ_K_BAD_LEN = 32,           /* a = length */
    FTLZ_K_EMPTY_BOOK = 33,
    FTLZ_K_KRAFT = 34,
    FTLZ_K_BITS_EXCEED = 35,
    FTLZ_K_SUMDC_LEN = 36,         /* a = raw_len */
    FTLZ_K_SUMDC_MISMATCH = 37,
    FTLZ_K_ORPHAN = 38,
    FTLZ_K_TRAILING = 39,          /* a = trailing byte count */
    FTLZ_K_RLE_ODD = 40,           /* "run-length stream has odd length" (encode.py:302-303), no offset */
    FTLZ_K_RLE_ZERO = 41,          /* "run-length stream has zero-length run" (encode.py:307-308) */
    /* decompression SDC detail (pipeline.py:565-577, encode.py:198-256) */
    FTLZ_K_D_PAST_END = 60,        /* "bit slice extends past payload end" */
    FTLZ_K_D_RAN_PAST = 61,        /* "code ran past block boundary" */
    FTLZ_K_D_OUTSIDE = 62,         /* "bit pattern outside Huffman code space" */
    FTLZ_K_D_CONSUMED = 63,        /* "block consumed {a} bits, expected {b}" */
    FTLZ_K_D_ZEROS = 64,           /* "block {block} decoded {a} unpredictable markers, record says {b}" */
    FTLZ_K_D_EMPTY = 65,           /* "empty block with nonzero bit length" */
    FTLZ_K_D_MISMATCH = 66         /* "block {block} mismatches after re-execution" */
};

/* `what` codes for FTLZ_K_TRUNCATED (container.py _Reader.take call sites) */
enum ftlz_field {
    FTLZ_F_HEADER = 0, FTLZ_F_INDICATOR = 1, FTLZ_F_COEFFS = 2, FTLZ_F_RECORD = 3,
    FTLZ_F_BOOK_SIZE = 4, FTLZ_F_BOOK_ENTRY = 5, FTLZ_F_PAYLOAD_LEN = 6, FTLZ_F_PAYLOAD = 7,
    FTLZ_F_UNPRED = 8, FTLZ_F_SUMDC_LENS = 9, FTLZ_F_SUMDC = 10
};

typedef struct ftlz_info {
    int32_t code;     /* ftlz_status */
    int32_t kind;     /* ftlz_kind   */
    int64_t offset;   /* CorruptStream offset, -1 if none */
    int64_t block;    /* block index, -1 if none */
    int64_t a, b;     /* message operands (see ftlz_kind) */
} ftlz_info;

/* FtConfig (pipeline.py:71-99) + QuantConfig (quantize.py:21-34) */
typedef struct ftlz_config {
    int32_t protect_input;
    int32_t protect_bins;
    int32_t duplicate_eval;
    int32_t store_sum_dc;
    int32_t block_edge;     /* 2..64, default 10 (core.py:18-20) */
    int32_t codec_id;       /* 0 identity, 1 run-length pairs; 2 (zlib) -> FTLZ_ERR_UNSUPPORTED_CODEC */
    uint32_t bin_capacity;  /* power of two >= 4, default 65536 */
    int32_t reserved;
} ftlz_config;

/* Fault-injection descriptor: replaces the process-global hooks seam (hooks.py:14-62) with
 * per-call data.  Semantics follow faults.py:157-189: XOR bit `bit` of one word. */
enum ftlz_fault_target {
    FTLZ_FAULT_INPUT = 0,    /* working input after stage (a) checksums   (STAGE_INPUT_AFTER_CHECKSUM) */
    FTLZ_FAULT_BINS = 1,     /* u32 bin word after stage (c)              (STAGE_BINS_FINALIZED)       */
    FTLZ_FAULT_DECOMP = 2,   /* decompressed word before verification, once (STAGE_DECOMP_BEFORE_VERIFY) */
    FTLZ_FAULT_COEFF = 3,    /* float32 regression coefficient `element` (STAGE_COEFFS_FITTED)        */
    FTLZ_FAULT_ESTIMATE = 4, /* float64 estimate: element 0 = e_reg, 1 = e_lor; bit 0..63 (STAGE_ESTIMATES) */
    /* duplicated evaluation (STAGE_DUP_EVAL, hooks.py:19, fired at pipeline.py:166-173): XOR one
     * bit of the float64 prediction / reconstruction of point `element` of `block` as evaluation
     * round r (1..3) returns it; `bit` = 64 * (r - 1) + b, b in 0..63.  Round 2 exists only with
     * duplicate_eval, round 3 only where rounds 1 and 2 disagree (2-of-3 vote). */
    FTLZ_FAULT_DUP_PREDICT = 5,
    FTLZ_FAULT_DUP_RECON = 6
};

typedef struct ftlz_fault {
    int32_t target;
    int32_t bit;
    int64_t block;
    int64_t element;   /* row-major offset inside the block (core.py:113-122) */
} ftlz_fault;

/* FtReport (pipeline.py:102-142).  Lists are caller-owned host arrays of `capacity` entries
 * (pass capacity >= number of blocks to never truncate); they come back sorted ascending. */
typedef struct ftlz_report {
    int64_t capacity;
    int64_t *input_corrected, *bins_corrected, *dup_mismatch, *reexecuted;
    int64_t n_input_corrected, n_bins_corrected, n_dup_mismatch, n_reexecuted;
    int32_t sdc;          /* decompression: terminal SDC, output withheld */
    int32_t reserved;
    ftlz_info info;       /* error detail when status != OK, or SDC detail when sdc != 0 */
    /* outputs describing the archive (compress) / stream (decompress) */
    double eb;            /* resolved absolute error bound */
    int64_t archive_len;
    int64_t n_blocks, n_regression, n_unpredictable, n_symbols, payload_bits;
    int32_t max_code_len;
    int32_t reserved2;
} ftlz_report;

/* Parsed 55-byte header (container.py:54, `<4sBBQQQIBdIQ`) */
typedef struct ftlz_header {
    int32_t version, codec_id;
    int64_t nx, ny, nz;
    int32_t block_edge, eb_mode;
    double eb_value;
    uint32_t bin_capacity;
    int32_t reserved;
    int64_t block_count;
} ftlz_header;

/* Section map of a validated archive (container.py:3-27) */
typedef struct ftlz_stream_info {
    ftlz_header hdr;
    int64_t table_off, table_len;      /* block table                         */
    int64_t book_off, n_symbols;       /* codebook: u32 count + 5 B entries   */
    int64_t payload_off, payload_len;  /* bytes after the u64 length          */
    int64_t unpred_off, n_unpred;      /* raw u32 words                       */
    int64_t sumdc_off;                 /* first of the 8 B sums, -1 if absent */
    int64_t n_regression, total_bits;
    int32_t max_code_len, has_sum_dc;
    /* stored (backend-coded) lengths: == payload_len and 8*nb for codec 0; for codec 1 the
     * run-length pair streams at payload_off / sumdc_off (payload_len is then the inverted length) */
    int64_t payload_stored_len, sumdc_stored_len;
} ftlz_stream_info;

/* ---- library identity ---------------------------------------------------------------------- */
int ftlz_abi_version(void);
const char* ftlz_last_error(void);   /* thread-local text of the last CUDA/argument failure */
void ftlz_default_config(ftlz_config* cfg);

/* ---- host-only helpers ----------------------------------------------------------------------- */
/* Header validation in the reference order (container.py:189-210). Returns FTLZ_OK or
 * FTLZ_ERR_CORRUPT_STREAM with `info` filled. */
int ftlz_peek_header(const uint8_t* h_data, size_t len, ftlz_header* hdr, ftlz_info* info);
/* ftlz_peek_header on a whole host archive of `len` bytes, plus the record-table bound: an
 * archive too short for the block records its header implies fails here with the reference's
 * CorruptStream kind and offset (container.py:212-218), before anything is sized by its dims. */
int ftlz_peek_archive(const uint8_t* h_data, size_t len, ftlz_header* hdr, ftlz_info* info);
/* Number of blocks of the partition (core.py:133-157), or -1 on invalid geometry. */
int64_t ftlz_block_count(int64_t nx, int64_t ny, int64_t nz, int32_t block_edge);

/* ---- stateless device API (caller-owned device memory; re-entrant across streams) ---------- */
size_t ftlz_compress_workspace_size(int64_t nx, int64_t ny, int64_t nz, const ftlz_config* cfg);
/* Upper bound of the archive size for these dims (worst case: every code 57 bits, every point
 * unpredictable).  The actual length is reported; FTLZ_ERR_CAPACITY if out_capacity is short. */
size_t ftlz_compress_bound(int64_t nx, int64_t ny, int64_t nz, const ftlz_config* cfg);
/* Compress a device-resident float32 field (row-major, dims nx*ny*nz) into a serialized
 * archive in d_out.  eb_mode: 0 = absolute, 1 = value-range relative (core.py:160-193).
 * faults / predictor_override are HOST arrays (override: nb int8, -1 = sampled choice,
 * 0 = Lorenzo, 1 = regression; pipeline.py:371-373).  Synchronises `stream` before return. */
int ftlz_compress(const float* d_in, int64_t nx, int64_t ny, int64_t nz,
                  int32_t eb_mode, double eb_value, const ftlz_config* cfg,
                  const ftlz_fault* faults, int64_t n_faults, const int8_t* predictor_override,
                  void* d_workspace, size_t workspace_size,
                  uint8_t* d_out, size_t out_capacity, ftlz_report* report, void* stream);

size_t ftlz_decompress_workspace_size(const ftlz_header* hdr, size_t archive_len);
/* Validate a device-resident archive (records, codebook, sections) without decoding.
 * `hdr` must come from ftlz_peek_header on the first 55 bytes. */
int ftlz_parse(const uint8_t* d_archive, size_t len, const ftlz_header* hdr,
               void* d_workspace, size_t workspace_size, ftlz_stream_info* info_out,
               ftlz_report* report, void* stream);
/* Decode + reconstruct + verify (+ one re-execution per mismatching block).  d_out holds
 * nx*ny*nz float32.  Returns FTLZ_OK with report->sdc set when the output must be withheld. */
int ftlz_decompress(const uint8_t* d_archive, size_t len, const ftlz_header* hdr,
                    float* d_out, const ftlz_fault* faults, int64_t n_faults,
                    void* d_workspace, size_t workspace_size, ftlz_report* report, void* stream);

/* ---- context API: the library owns device workspaces, pinned staging and a stream -------- */
typedef struct ftlz_ctx ftlz_ctx;
ftlz_ctx* ftlz_ctx_create(int32_t device);
void ftlz_ctx_destroy(ftlz_ctx* ctx);
void* ftlz_ctx_stream(ftlz_ctx* ctx);
/* device input -> archive kept in the context (ftlz_ctx_archive_device) */
int ftlz_ctx_compress_device(ftlz_ctx* ctx, const float* d_in, int64_t nx, int64_t ny, int64_t nz,
                             int32_t eb_mode, double eb_value, const ftlz_config* cfg,
                             const ftlz_fault* faults, int64_t n_faults,
                             const int8_t* predictor_override, ftlz_report* report);
/* host input (pinned or pageable) -> archive copied to the context's pinned buffer */
int ftlz_ctx_compress_host(ftlz_ctx* ctx, const float* h_in, int64_t nx, int64_t ny, int64_t nz,
                           int32_t eb_mode, double eb_value, const ftlz_config* cfg,
                           const ftlz_fault* faults, int64_t n_faults,
                           const int8_t* predictor_override, ftlz_report* report);
/* as ftlz_ctx_compress_host, with the archive downloaded straight into h_out (e.g. pinned
 * memory): no staging copy.  FTLZ_ERR_CAPACITY (report->archive_len set, archive kept on the
 * device for ftlz_ctx_copy_archive) when out_capacity is too small. */
int ftlz_ctx_compress_host_to(ftlz_ctx* ctx, const float* h_in, int64_t nx, int64_t ny, int64_t nz,
                              int32_t eb_mode, double eb_value, const ftlz_config* cfg,
                              const ftlz_fault* faults, int64_t n_faults, const int8_t* predictor_override,
                              uint8_t* h_out, size_t out_capacity, ftlz_report* report);
int ftlz_ctx_archive_device(ftlz_ctx* ctx, const uint8_t** d_ptr, size_t* len);
int ftlz_ctx_archive_host(ftlz_ctx* ctx, const uint8_t** h_ptr, size_t* len);
/* copy the last archive into caller memory (host) */
int ftlz_ctx_copy_archive(ftlz_ctx* ctx, void* h_dst, size_t capacity);
/* host archive -> device validation; the validated device copy is kept for decompression */
int ftlz_ctx_parse_host(ftlz_ctx* ctx, const uint8_t* h_archive, size_t len,
                        ftlz_stream_info* info_out, ftlz_report* report);
/* host archive -> host float32 output (h_out: nx*ny*nz floats, pinned or pageable).
 * If `reuse_parsed` is nonzero and the same archive was just parsed, the upload is skipped.
 * Large fields are decoded in slabs whose output is downloaded while later slabs decode, so
 * h_out is unspecified when report->sdc withholds the output. */
int ftlz_ctx_decompress_host(ftlz_ctx* ctx, const uint8_t* h_archive, size_t len, float* h_out,
                             const ftlz_fault* faults, int64_t n_faults, int32_t reuse_parsed,
                             ftlz_report* report);
/* region extraction (pipeline.py:726-795): only the blocks intersecting the half-open box
 * region = {x0, y0, z0, x1, y1, z1} are decoded, reconstructed and verified (one re-execution);
 * h_out receives (x1-x0)*(y1-y0)*(z1-z0) float32 values, bit-identical to the same slice of a
 * full decompression.  FTLZ_ERR_INVALID_REGION when the box is empty or outside the dims. */
int ftlz_ctx_decompress_region_host(ftlz_ctx* ctx, const uint8_t* h_archive, size_t len, const int64_t* region,
                                    float* h_out, int32_t reuse_parsed, ftlz_report* report);
/* blocks a region extraction decodes (pipeline.py:798-810) */
int64_t ftlz_intersecting_block_count(int64_t nx, int64_t ny, int64_t nz, int32_t block_edge, const int64_t* region);
/* backend codec 1 (encode.py:287-312) on the device for host bytes: invert == 0 applies the
 * run-length pairs, invert != 0 inverts them (FTLZ_ERR_CORRUPT_STREAM, kind FTLZ_K_RLE_ODD /
 * FTLZ_K_RLE_ZERO, on a malformed stream).  *out_len receives the result length; when it
 * exceeds `capacity` nothing usable is written and FTLZ_ERR_CAPACITY is returned (retry with
 * a larger buffer).  serialize / stream materialisation use it for codec-1 streams. */
int ftlz_ctx_rle_host(ftlz_ctx* ctx, const uint8_t* h_in, size_t n, int32_t invert, uint8_t* h_out,
                      size_t capacity, size_t* out_len, ftlz_info* info);
/* device archive -> device output */
int ftlz_ctx_decompress_device(ftlz_ctx* ctx, const uint8_t* d_archive, size_t len,
                               const ftlz_header* hdr, float* d_out,
                               const ftlz_fault* faults, int64_t n_faults, ftlz_report* report);

/* ---- instrumentation (bench.py): per-kernel CUDA-event timing on the context stream ------- */
int ftlz_ctx_profile(ftlz_ctx* ctx, int32_t enable);   /* enable/disable and reset totals */
/* up to max_n kernels: '\n'-separated names, accumulated ms and launch counts; returns count */
int ftlz_ctx_profile_read(ftlz_ctx* ctx, char* names, size_t names_cap, double* ms, int64_t* counts,
                          int32_t max_n);

#ifdef __cplusplus
}
#endif
#endif /* FTLZ_B200_H */
