/*
 * qrmark_gpu.h — C-ABI of the B200-native QRMark tile-detection path.
 *
 * This is the drop-in boundary: plain C types, plain pointers and sizes, no
 * C++ or torch types. Each entry point names the reference interface it
 * replaces (paths relative to /root/reference/proj). The C++ drop-in API
 * (include/qrmark/<module>.hpp, namespace qrmark) and the Python package
 * (paper_2509_02447_b200) are both thin layers over these calls.
 *
 * Conventions
 *  - Status codes only; no exception crosses the ABI. The C++ layer maps
 *    QRM_INVALID_INPUT / QRM_DIVISION_BY_ZERO / QRM_INFEASIBLE back to the
 *    reference exceptions (include/qrmark/errors.hpp:11-25). qrm_last_error()
 *    returns the message of the calling thread's last failure.
 *  - Packed words: a codeword / message of <= 64 bits is a uint64_t holding bit
 *    0 of the reference BitVec (rs.hpp:16) in its most significant used bit,
 *    i.e. word = sum_b bit[b] << (nbits-1-b). Symbols are MSB-first m-bit
 *    groups (rs.cpp:8-25).
 *  - "_device" calls take device pointers and a cudaStream_t passed as void*
 *    (NULL = legacy default stream); they are stream-ordered and asynchronous.
 *    "_host" calls take host pointers and return when results are in host
 *    memory.
 *  - One context per device and host thread; a context is not thread-safe.
 *  - There is no CPU fallback: every compute call runs on the GPU and fails
 *    with QRM_CUDA_ERROR / QRM_NO_DEVICE when it cannot.
 */
#ifndef QRMARK_GPU_H
#define QRMARK_GPU_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#if defined(__GNUC__)
#define QRM_EXPORT __attribute__((visibility("default")))
#else
#define QRM_EXPORT
#endif

typedef enum qrm_status {
    QRM_OK = 0,
    QRM_INVALID_INPUT = 1,    /* qrmark::InvalidInput    (errors.hpp:11) */
    QRM_DIVISION_BY_ZERO = 2, /* qrmark::DivisionByZero  (errors.hpp:16) */
    QRM_INFEASIBLE = 3,       /* qrmark::InfeasibleConfig (errors.hpp:22) */
    QRM_CUDA_ERROR = 4,
    QRM_NO_DEVICE = 5,
    QRM_INTERNAL = 6
} qrm_status;

/* TileStrategy (tiling.hpp:13) */
enum { QRM_TILE_RANDOM = 0, QRM_TILE_RANDOM_GRID = 1, QRM_TILE_FIXED = 2 };

/* Record status */
enum { QRM_REC_FAILED = 0, QRM_REC_DECODED = 1 };

/* DetectionConfig (detect.hpp:25-37) + CodeParams (rs.hpp:26-37). */
typedef struct qrm_config {
    int symbol_bits;            /* m: 4 (GF(16), poly 0x13) or 8 (GF(256), poly 0x11D) */
    int n, k;                   /* code length / dimension, X_i = alpha^i (rs.cpp:52-63) */
    int tile_size;              /* l (TileSpec::size, tiling.hpp:16-20) */
    int tile_strategy;          /* QRM_TILE_* */
    uint64_t tile_seed;         /* TileSpec::seed */
    uint64_t key_seed;          /* WatermarkKey::seed (stego.hpp:15-19) */
    double alpha;               /* WatermarkKey::alpha */
    const uint8_t* key_message; /* k*m bits, one 0/1 byte per bit (host memory) */
    double fpr_target;          /* DetectionConfig::fpr_target */
} qrm_config;

/* DetectionRecord (detect.hpp:45-55), compact device form. bit_acc =
 * matches / (n*m); corrected present iff status == QRM_REC_DECODED. */
typedef struct qrm_record {
    uint64_t raw;      /* hardened extractor output m' (packed) */
    uint64_t msg;      /* RS-corrected information bits c_s (packed), 0 on failure */
    uint8_t status;    /* QRM_REC_* */
    uint8_t errors;    /* errors_corrected (0 on failure) */
    uint8_t matches;   /* raw vs key codeword matching bits */
    uint8_t verified;  /* detect.cpp:186-195 */
    uint8_t ties;      /* correlations that were exactly zero (resolved bit-exactly) */
    uint8_t reserved[3];
} qrm_record;

/* StreamPlan (sched.hpp:26-34) for the 3-stage host pipeline. */
typedef struct qrm_plan {
    int streams[3];   /* s[k]: transfer / decode / correct+return */
    int minibatch[3]; /* m[k] */
} qrm_plan;

/* Per-call stage timings of qrm_detect_host (cudaEvent based, ms). */
typedef struct qrm_host_stats {
    double wall_ms;
    double h2d_bytes;
    double d2h_bytes;
    int minibatches;
    int kernel_launches;
} qrm_host_stats;

/* SyntheticStageLoad (detect.hpp:127-131): extra work per image in each
 * stage (preprocess / extract / correct in the reference; transfer / decode /
 * correct+return here). The reference sleeps ns per item in each worker
 * (detect.cpp:243-245, 304, 318, 336); here each mini-batch of b images on a
 * stage's stream is held for b * ns by a device-side wait on that stream, so
 * s concurrent streams of a stage model s workers, as in the reference. */
typedef struct qrm_stage_load {
    int64_t ns[3];
} qrm_stage_load;

/* DeskReport / StageLatencies accounting (detect.hpp:39-43, 134-139) of one
 * host-pipeline call, from cudaEvents on the stage streams (plus the host
 * gather time of the staged transfer): busy_ns[k] = sum over mini-batches of
 * stage k's span; image_ns (nullable, caller-owned count x 3) = the stage spans
 * of each image's mini-batch (every image of a mini-batch is in flight for the
 * whole span). */
typedef struct qrm_stage_times {
    int64_t wall_ns;
    int64_t busy_ns[3];
    int64_t* image_ns;
} qrm_stage_times;

typedef struct qrm_ctx qrm_ctx;

QRM_EXPORT const char* qrm_last_error(void);
QRM_EXPORT int qrm_abi_version(void);
QRM_EXPORT int qrm_device_count(void);
/* Host CPUs on the NUMA node of GPU `device` (sysfs local_cpulist of its PCI
 * function): *count of them, the first `capacity` written to cpus. *count = 0
 * when unknown. The multi-GPU host executor pins each shard's host thread (and
 * each context's staging workers) to these CPUs. */
QRM_EXPORT qrm_status qrm_device_cpus(int device, int* cpus, int capacity, int* count);

/* ---------------------------------------------------------------- context
 * Replaces DetectionContext::DetectionContext (detect.cpp:135-146) and the
 * SpreadSpectrumCodec constructor (stego.cpp:16-27): validates the config,
 * builds the +-1 pattern planes on the device, the GF tables, the key
 * codeword (rs_encode, rs.cpp:78-91) and the verify thresholds
 * (verify_threshold, detect.cpp:31-66). */
QRM_EXPORT qrm_status qrm_ctx_create(int device, const qrm_config* cfg, qrm_ctx** out);
QRM_EXPORT void qrm_ctx_destroy(qrm_ctx* ctx);
/* Key codeword (packed) and thresholds tau(k*m), tau(n*m) of the context. */
QRM_EXPORT qrm_status qrm_ctx_info(const qrm_ctx* ctx, uint64_t* key_codeword, uint64_t* key_message, int* tau_msg,
                                   int* tau_raw);

/* ----------------------------------------------------------------- detect
 * Replaces detect_batch (detect.cpp:250-368) / DetectionContext::detect_one
 * (detect.cpp:164-198) for a uniform batch: `count` images of w x h RGB u8,
 * interleaved HWC (image.hpp:28-30), image i at images + i*image_stride.
 * draw_index of image i = first_draw + i (tiling.cpp:40). Device-resident:
 * `images` and `out` are device pointers (or mapped pinned host memory). */
QRM_EXPORT qrm_status qrm_detect_device(qrm_ctx* ctx, const uint8_t* images, int64_t count, int w, int h,
                                        int64_t image_stride, uint64_t first_draw, qrm_record* out, void* stream);

/* Stream overlap of qrm_detect_device. The decode kernel is launched with
 * programmatic dependent launch: by default (enable = 0) it reads no window
 * before the preceding kernel on the stream has completed, so the images may
 * be produced by any kernel just before the call. enable = 1 is the caller's
 * promise that the images are complete before the preceding kernel on the
 * stream runs (e.g. a resident batch decoded back to back): the window loads
 * then overlap the previous decode's tail. Records are identical either way. */
QRM_EXPORT qrm_status qrm_ctx_set_input_overlap(qrm_ctx* ctx, int enable);

/* Same, from HOST images to HOST records, through the stream pipeline (the
 * CUDA-stream executor that replaces detect_batch's thread pools and bounded
 * queues). plan == NULL uses the context's current plan (qrm_ctx_set_plan).
 * mode 0: window-only transfer (the tile window is read from mapped pinned host
 * memory by the decode kernel); mode 1: full-image H2D copies; mode 2: staged
 * window transfer (a host worker pool copies each image's l x l window into
 * pinned staging, one contiguous H2D per mini-batch); mode 3: both at once on
 * each mini-batch -- a share (qrm_ctx_set_transfer_split, default 0.5) of the
 * windows fetched zero-copy while the workers stage the rest for the copy
 * engine. Host images are registered (page-locked) for the call if they are
 * not pinned already. */
QRM_EXPORT qrm_status qrm_detect_host(qrm_ctx* ctx, const uint8_t* images, int64_t count, int w, int h,
                                      int64_t image_stride, uint64_t first_draw, qrm_record* out,
                                      const qrm_plan* plan, int mode, qrm_host_stats* stats);

/* qrm_detect_host with the reference's SyntheticStageLoad and DeskReport stage
 * accounting (both nullable). */
QRM_EXPORT qrm_status qrm_detect_host_timed(qrm_ctx* ctx, const uint8_t* images, int64_t count, int w, int h,
                                            int64_t image_stride, uint64_t first_draw, qrm_record* out,
                                            const qrm_plan* plan, int mode, const qrm_stage_load* load,
                                            qrm_stage_times* times);

/* detect_batch over a std::span<const ImageBuffer> (detect.cpp:250-368): `count`
 * same-size w x h images at separate, pageable host addresses images[i] (each
 * ImageBuffer's own bytes; nothing is registered or copied whole). The staged
 * transfer (mode 2) moves only each image's l x l window: the context's host
 * workers gather the windows into a context-owned pinned staging ring that the
 * copy engine moves to the device while the next piece is gathered. Needs
 * min(w, h) >= 256 (inputs that need the bilinear upscale take
 * qrm_detect_ragged). load / times as qrm_detect_host_timed. */
QRM_EXPORT qrm_status qrm_detect_host_images(qrm_ctx* ctx, const uint8_t* const* images, int64_t count, int w,
                                             int h, uint64_t first_draw, qrm_record* out, const qrm_plan* plan,
                                             const qrm_stage_load* load, qrm_stage_times* times);

/* Ragged batch (std::span<const ImageBuffer> of mixed sizes, detect.hpp:145):
 * per-image host pointers and sizes. Images smaller than 256 px take the
 * bilinear upscale path (transforms.cpp:24-47). */
QRM_EXPORT qrm_status qrm_detect_ragged(qrm_ctx* ctx, const uint8_t* const* images, const int* widths,
                                        const int* heights, int64_t count, uint64_t first_draw, qrm_record* out);

/* SpreadSpectrumCodec::extract + harden (stego.cpp:10-14, 53-67) for a
 * uniform device batch: soft (count x n*m doubles, nullable) and raw words.
 * soft_i = S_i / (255 * 3 l^2) with S_i the exact integer correlation. */
QRM_EXPORT qrm_status qrm_extract_device(qrm_ctx* ctx, const uint8_t* images, int64_t count, int w, int h,
                                         int64_t image_stride, uint64_t first_draw, double* soft, uint64_t* raw,
                                         void* stream);

/* The learned extractor behind the WatermarkCodec plug-in point
 * (stego.hpp:32-40): a HiDDeN / Stable-Signature-style conv stack (9 x conv3x3
 * + BN + ReLU at 64x64, avg-pool, linear; contract in oracle/hidden_oracle.c)
 * with random-init weights drawn from `weight_seed`, run as implicit-GEMM
 * tcgen05 bf16 kernels, then the same RS correction and verify as
 * qrm_detect_device. logits (count x n*m floats) is nullable. Needs l = 64. */
QRM_EXPORT qrm_status qrm_hidden_detect_device(qrm_ctx* ctx, const uint8_t* images, int64_t count, int w, int h,
                                               int64_t image_stride, uint64_t first_draw, uint64_t weight_seed,
                                               float* logits, qrm_record* out, void* stream);

/* qrm_detect_host with Algorithm 2 (resource-aware mini-batch scheduling,
 * PAPER.md 6.2; lpt_schedule, sched.cpp:177-235) choosing the decode stream of
 * every mini-batch: tasks are the plan's mini-batches, their latencies the
 * decode time per image of this context's last qrm_warmup_profile(_mode)
 * (uniform when none ran); LPT with balance slack lambda shards tasks into
 * b_min-image pieces where needed. Records are identical to qrm_detect_host. */
QRM_EXPORT qrm_status qrm_detect_host_lpt(qrm_ctx* ctx, const uint8_t* images, int64_t count, int w, int h,
                                          int64_t image_stride, uint64_t first_draw, qrm_record* out,
                                          const qrm_plan* plan, int mode, double lambda, int b_min,
                                          qrm_host_stats* stats);

/* qrm_detect_host over several contexts (normally one per device of the node,
 * SURVEY 8e): context i decodes the contiguous shard [count*i/n,
 * count*(i+1)/n) with its global draw indices on its own host thread, and its
 * records land at their global positions in `out`. Images are independent, so
 * there is no collective; the result equals one qrm_detect_host over the whole
 * batch. stats (nullable) sums the shards' bytes and launches. */
QRM_EXPORT qrm_status qrm_detect_host_multi(qrm_ctx* const* ctxs, int nctx, const uint8_t* images, int64_t count,
                                            int w, int h, int64_t image_stride, uint64_t first_draw, qrm_record* out,
                                            const qrm_plan* plan, int mode, qrm_host_stats* stats);

/* Tile extraction + normalisation (north-star item 1): for each image,
 * preprocess (transforms.cpp:42-47) -> select_tile (draw first_draw + i,
 * tiling.cpp:23-47) -> extract_tile (tiling.cpp:62-77) -> normalize
 * (image.cpp:32-38), emitted as bf16 NHWC [count][64][64][channels]
 * (channels 3, or 4 with a zero 4th channel for 8-byte pixels) in device
 * memory: the input a learned decoder's first layer consumes. Needs l = 64. */
QRM_EXPORT qrm_status qrm_extract_tiles_device(qrm_ctx* ctx, const uint8_t* images, int64_t count, int w, int h,
                                               int64_t image_stride, uint64_t first_draw, int channels, void* out,
                                               void* stream);

/* Diagnostics for the learned extractor's per-layer checks
 * (scripts/debug_hidden_layers.py): runs conv layers 0..stop_after on a device
 * batch and copies that layer's output to `out` -- bf16 NHWC
 * [count][64][64][64] activations, or for the last layer (stop_after = 8) the
 * fp32 per-block channel sums [count][32][64]. */
QRM_EXPORT qrm_status qrm_hidden_debug_activation(qrm_ctx* ctx, const uint8_t* images, int64_t count, int w, int h,
                                                  int64_t image_stride, uint64_t first_draw, uint64_t weight_seed,
                                                  int stop_after, void* out, void* stream);

/* Extractor behind the WatermarkCodec plug-in point (stego.hpp:32-40) used by
 * qrm_detect_device / qrm_detect_host / qrm_detect_ragged:
 *   QRM_EXTRACTOR_SPREAD_SPECTRUM (default): SpreadSpectrumCodec::extract
 *     (stego.cpp:53-67), the reference's own extractor;
 *   QRM_EXTRACTOR_CONV: the learned conv stack of qrm_hidden_detect_device
 *     with weights drawn from weight_seed (needs tile_size 64).
 * RS correction, verify and the record layout are the same for both. */
#define QRM_EXTRACTOR_SPREAD_SPECTRUM 0
#define QRM_EXTRACTOR_CONV 1
QRM_EXPORT qrm_status qrm_ctx_set_extractor(qrm_ctx* ctx, int kind, uint64_t weight_seed);

/* Host pipeline mode 3: the share of each mini-batch's windows the transfer
 * kernel fetches zero-copy; the rest go through pinned staging and the copy
 * engine. Both paths give the same records. */
QRM_EXPORT qrm_status qrm_ctx_set_transfer_split(qrm_ctx* ctx, double zero_copy_fraction);

/* ---- robustness attacks -------------------------------- */

/* TransformOp (transforms.hpp:22-35), in the reference's order. */
enum {
    QRM_ATTACK_CENTERCROP = 0, QRM_ATTACK_RESIZETO, QRM_ATTACK_NORMALIZE, QRM_ATTACK_CROP, QRM_ATTACK_RESIZE,
    QRM_ATTACK_BRIGHTNESS, QRM_ATTACK_CONTRAST, QRM_ATTACK_SATURATION, QRM_ATTACK_SHARPNESS, QRM_ATTACK_BLUR,
    QRM_ATTACK_OVERLAY_TEXT, QRM_ATTACK_JPEG_APPROX
};
/* apply_attack (transforms.cpp:289-362) on `count` same-size byte images in
 * device memory (image i at images + i*image_stride), bit-exact with the
 * reference. Output sizes depend on the op: out == NULL only reports them in
 * *out_w / *out_h. Results go to out + i*out_stride (bytes; NORMALIZE writes
 * floats). Parameter checks and messages are the reference's (InvalidInput).
 * Stream-ordered; temporaries are freed before return. */
QRM_EXPORT qrm_status qrm_attack_device(const uint8_t* images, int64_t count, int w, int h, int64_t image_stride,
                                        int op, double param, void* out, int64_t out_stride, int* out_w, int* out_h,
                                        void* stream);

/* ---- formats either side of the path (ingest and report) ---------------- */

/* read_ppm (image.cpp:129-146): P6, maxval 255, '#' comments, the reference's
 * InvalidInput messages. dst == NULL: header only (w, h). Else the raster
 * (w*h*3 bytes, HWC) goes to dst, which must hold cap >= w*h*3 bytes. */
QRM_EXPORT qrm_status qrm_ppm_read(const char* path, uint8_t* dst, int64_t cap, int* w, int* h);
/* write_ppm (image.cpp:148-156). */
QRM_EXPORT qrm_status qrm_ppm_write(const char* path, const uint8_t* img, int w, int h);
/* ingest (cli.cpp:22-45) of `count` same-size P6 files, decoded in parallel by
 * `threads` host threads straight into dst + i*image_stride (typically pinned
 * memory that qrm_detect_host then transfers). status[i] (nullable) per file;
 * returns the first failure. */
QRM_EXPORT qrm_status qrm_ppm_read_batch(const char* const* paths, int64_t count, int w, int h, uint8_t* dst,
                                         int64_t image_stride, int threads, int32_t* status);
/* DetectionRecord::cache_hit: the CorrectionCache policy (detect.cpp:86-128;
 * capacity / stale_after of CacheConfig, detect.hpp:19-23) replayed over the
 * records' raw words in index order (the reference with one correct worker).
 * The GPU decoders are O(1) per word, so the codebook is never consulted for
 * speed; this reproduces the flag the reference reports. hit: count bytes. */
QRM_EXPORT qrm_status qrm_cache_hits(const qrm_record* records, int64_t count, int64_t capacity,
                                     uint64_t stale_after, uint8_t* hit);
/* The "records" array of cmd_detect's report (cli.cpp:279-281): record_to_json
 * (json_io.cpp:98-120, deterministic stage times) of every record, in
 * nlohmann::json dump(2) layout. Index of record i = first_index + i.
 * cache_hit replays CorrectionCache (detect.cpp:86-128; CacheConfig
 * detect.hpp:19-23: enabled, capacity, stale_after) over the records in index
 * order. Writes at most cap-1 bytes + NUL to out (nullable); *len = the full
 * length. */
QRM_EXPORT qrm_status qrm_records_json(const qrm_record* records, int64_t count, int n_bits, int k_bits,
                                       int64_t first_index, int cache_enabled, int64_t cache_capacity,
                                       uint64_t stale_after, char* out, int64_t cap, int64_t* len);

/* preprocess (transforms.cpp:42-47) of one host image -> 256*256*3 floats. */
QRM_EXPORT qrm_status qrm_preprocess_host(const uint8_t* image, int w, int h, float* out);

/* General window resample of one host byte image on the device: pixel
 * (x + x_off, y + y_off) of the image bilinearly resized to sw x sh
 * (resize_bilinear, image.cpp:57-85; upscale = 0: the image itself), for an
 * out_w x out_h window; u8 out, or float(v/127.5 - 1) (normalize,
 * image.cpp:32-38) when normalize != 0. Covers resize_bilinear, center_crop
 * (image.cpp:87-105), extract_tile (tiling.cpp:62-77) and preprocess. */
QRM_EXPORT qrm_status qrm_resample_host(const uint8_t* image, int w, int h, int upscale, int sw, int sh, int x_off,
                                        int y_off, int out_w, int out_h, int normalize, void* out);

/* SpreadSpectrumCodec::extract (stego.cpp:53-67) of one normalised float tile
 * (3 l^2 floats, any values): the reference's sequential double summation
 * replayed on the device -> bit-identical soft values. */
QRM_EXPORT qrm_status qrm_extract_float_host(uint64_t key_seed, int n_bits, int l, const float* tile, double* soft);

/* ----------------------------------------------------------------- RS
 * Replace bw_decode (rs.cpp:188-196), bit-exact: the unique codeword within
 * distance t or failure. nerr_out[i] = errors_corrected, or -1 for a decode
 * failure (nullopt). */
/* Packed words (n*m <= 64). algo 0: auto; 1: thread-per-codeword syndrome
 * decoder (t = 1 codes); 2: segmented-warp Berlekamp-Massey/Chien/Forney (4
 * lanes per codeword, any t <= 8); 3: algo 2 behind the device codebook (the
 * CorrectionCache analog, detect.cpp:86-128: a per-(device, code) memo of
 * decoded words, n*m < 64; results are identical with or without it). */
QRM_EXPORT qrm_status qrm_rs_decode_packed_device(int m, int n, int k, const uint64_t* words, int64_t count,
                                                  uint64_t* cw_out, int8_t* nerr_out, int algo, void* stream);
/* Symbol arrays (any n <= 2^m - 1, m in {4, 8}): count*n bytes in/out. */
/* Empty the device codebook of code (m, n, k) on the current device. */
QRM_EXPORT qrm_status qrm_rs_codebook_clear(int m, int n, int k, void* stream);
QRM_EXPORT qrm_status qrm_rs_decode_symbols_device(int m, int n, int k, const uint8_t* recv, int64_t count,
                                                   uint8_t* cw_out, int8_t* nerr_out, void* stream);
/* RS stress words (SURVEY 8d recipe) on the device: per word a random message,
 * its codeword with e injected symbol errors (e <= t for 90%, t+1..3 for 10%). */
QRM_EXPORT qrm_status qrm_rs_stress_device(int m, int n, int k, uint64_t seed, int64_t count, uint64_t* msg,
                                           uint64_t* words, int8_t* nerr_true, void* stream);
/* RS stress words for symbol codes (any n <= 255, m <= 8, k*(n-k) <= 96 KiB):
 * per word the codeword of a random message (true_cw, [count][n] symbols),
 * the received word with e injected symbol errors (recv) and e (nerr_true);
 * e <= t for 90% of words, t+1..t+2 for 10%. */
QRM_EXPORT qrm_status qrm_rs_stress_symbols_device(int m, int n, int k, uint64_t seed, int64_t count,
                                                   uint8_t* true_cw, uint8_t* recv, int8_t* nerr_true, void* stream);
/* rs_encode (rs.cpp:78-91) on the host, packed (n*m <= 64). */
QRM_EXPORT qrm_status qrm_rs_encode_packed(int m, int n, int k, uint64_t message, uint64_t* codeword);
/* verify_threshold (detect.cpp:31-66). */
QRM_EXPORT qrm_status qrm_verify_threshold(int n_bits, double fpr, int* tau);

/* ----------------------------------------------------------------- inputs
 * Synthetic corpus on the device (cmd_bench recipe, cli.cpp:404-411):
 * image i = synthetic_image(first_seed + i, w, h) (image.cpp:157-189),
 * optionally normalize -> embed_image_grid (stego.cpp:77-92) with the key
 * codeword -> denormalize. Output u8 [count][h][w][3] at `out` (device). */
QRM_EXPORT qrm_status qrm_make_corpus_device(const qrm_config* cfg, uint64_t first_seed, int64_t count, int w,
                                             int h, int embed, uint8_t* out, void* stream);
/* The codec's +-1 planes (stego.cpp:22-26), n_bits x 3l^2 int8 (device). */
QRM_EXPORT qrm_status qrm_patterns_device(uint64_t key_seed, int n_bits, int l, int8_t* out, void* stream);

/* ------------------------------------------------------------- scheduler
 * allocate_streams (sched.cpp:50-114): Algorithm 1. */
QRM_EXPORT qrm_status qrm_allocate_streams(int stages, const double* time, const double* memory, double b0,
                                           int global_batch, int stream_budget, double m_cap, double epsilon,
                                           int stall_cap, int* streams_out, int* minibatch_out,
                                           double* bottleneck_out);
/* Algorithm 1 with a GPU-aware stage model (extension; not in the reference):
 * TIME(k, s, m) = t[k] (m / b0) / min(s, sat[k]), sat[k] the measured speedup
 * of stage k on concurrent streams (qrm_warmup_saturation). With every sat[k]
 * >= stream_budget this is qrm_allocate_streams. */
QRM_EXPORT qrm_status qrm_allocate_streams_sat(int stages, const double* time, const double* memory,
                                               const double* sat, double b0, int global_batch, int stream_budget,
                                               double m_cap, double epsilon, int stall_cap, int* streams_out,
                                               int* minibatch_out, double* bottleneck_out);
/* lpt_schedule (sched.cpp:177-235): Algorithm 2. Pieces are returned stream
 * by stream in placement order. */
QRM_EXPORT qrm_status qrm_lpt_schedule(int ntasks, const int* ids, const double* latency, const double* memory,
                                       const int* units, int stream_count, double lambda, double m_cap, int b_min,
                                       int global_batch, int capacity, int* p_stream, int* p_id, int* p_units,
                                       double* p_latency, double* p_memory, int* p_mb, int* n_pieces,
                                       double* loads, int* m_unit);
/* warmup_profile (sim.cpp:240-288): cudaEvent-timed warm-up of the three
 * device stages (transfer, decode, correct) at baseline batch b0 on `images`
 * (host, uniform w x h). Fills time[3] (ms per b0 images), memory[3] (bytes
 * per image). */
QRM_EXPORT qrm_status qrm_warmup_profile(qrm_ctx* ctx, const uint8_t* images, int64_t count, int w, int h,
                                         int64_t image_stride, int warmup_iters, int b0, double* time,
                                         double* memory);
/* GPU-aware warm-up (extension): the mode-0 stages (window fetch, decode,
 * record D2H) each on 1, 2 and 4 concurrent streams of b0 images (host images,
 * count >= 4 b0). time[3] = ms per b0 images on one stream, memory[3] bytes
 * per image, sat[3] = best speedup s T(1) / T(s) (1 = no gain from streams;
 * speedups under 10 % count as none, being within run-to-run noise). */
QRM_EXPORT qrm_status qrm_warmup_saturation(qrm_ctx* ctx, const uint8_t* images, int64_t count, int w, int h,
                                            int64_t stride, int iters, int b0, double* time, double* memory,
                                            double* sat);
/* As qrm_warmup_profile with the transfer stage of host-pipeline mode `mode`
 * (0: zero-copy window fetch, memory[0] = 3 l^2 B/image; 1: full-image copy). */
QRM_EXPORT qrm_status qrm_warmup_profile_mode(qrm_ctx* ctx, const uint8_t* images, int64_t count, int w, int h,
                                              int64_t image_stride, int iters, int b0, int mode, double* time,
                                              double* memory);
/* Sets the plan used by qrm_detect_host when its plan argument is NULL. */
QRM_EXPORT qrm_status qrm_ctx_set_plan(qrm_ctx* ctx, const qrm_plan* plan);

/* Measurement hook: runs the device detect path `reps` times on a uniform
 * device batch and returns the mean duration of the decode kernel alone
 * (cudaEvents recorded on its stream immediately around each launch). */
QRM_EXPORT qrm_status qrm_probe_decode_kernel(qrm_ctx* ctx, const uint8_t* images, int64_t count, int w, int h,
                                              int64_t image_stride, int reps, double* avg_ms);

/* Number of kernels this library has launched in the calling process. */
QRM_EXPORT uint64_t qrm_kernel_launch_count(void);

#ifdef __cplusplus
}
#endif

#endif /* QRMARK_GPU_H */
