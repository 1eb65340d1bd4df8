// C-ABI implementation (include/qrmark_gpu.h): context, device-resident and
// host-buffer detection, RS batch decode, corpus generation, planners.
//
// The host-buffer path (qrm_detect_host) is the CUDA-stream executor that
// replaces detect_batch's three thread pools and bounded queues
// (detect.cpp:250-368): the batch is cut into mini-batches that flow through
// three stages — transfer (H2D copy engine, or nothing when the decode kernel
// reads the tile window straight out of mapped pinned host memory), decode
// (tcgen05 correlation + fused harden/RS/verify) and correct/return (tie /
// general-t completion kernel + D2H of the compact records) — with stage k
// round-robining its mini-batches over plan.streams[k] CUDA streams and
// cudaEvents instead of queues between stages.
#include <cuda_runtime.h>
#include <pthread.h>
#include <sched.h>

#include <algorithm>
#include <immintrin.h>
#include <atomic>
#include <chrono>
#include <cmath>
#include <cstring>
#include <fstream>
#include <map>
#include <memory>
#include <mutex>
#include <string>
#include <tuple>
#include <thread>
#include <vector>

#include "host_code.hpp"
#include "qrm_device.cuh"
#include "qrm_types.h"
#include "qrmark_gpu.h"
#include <cudaTypedefs.h>
#include <nvtx3/nvToolsExt.h>

#include "host_pool.hpp"
#include "qrm_hidden.h"
#include "sched_host.hpp"

namespace qrm {
cudaError_t launch_corr_detect(const DetectParams& p, int sm_count, cudaStream_t st);
cudaError_t launch_detect_finish(const DetectParams& p, int tmax, int sm_count, cudaStream_t st);
cudaError_t launch_gather_windows(const GatherDesc* descs, int64_t count, int l, uint8_t* out, cudaStream_t st);
cudaError_t launch_fetch_windows(const WindowSource& src, int64_t count, int K, uint8_t* out, int sm_count,
                                 cudaStream_t st);
cudaError_t launch_fetch_windows_tma(const CUtensorMap& tmap, const WindowSource& src, int64_t count, uint8_t* out,
                                     int sm_count, cudaStream_t st);
cudaError_t launch_attack_pixels(const AttackParams& p, cudaStream_t st);
cudaError_t launch_tile_bf16(const CUtensorMap& tmap, const TileBf16Params& p, int sm_count, cudaStream_t st);
cudaError_t launch_attack_jpeg(const AttackParams& p, cudaStream_t st);
cudaError_t launch_attack_resample(const AttackParams& p, cudaStream_t st);
cudaError_t launch_rs_packed(const RsTables* tab, int m, int n, int r, int t, int algo, const uint64_t* words,
                             int64_t count, uint64_t* cw, int8_t* nerr, int sm_count, cudaStream_t st,
                             CodebookTable cache);
cudaError_t launch_rs_symbols(const RsTables* tab, int n, int t, const uint8_t* recv, int64_t count, uint8_t* cw,
                              int8_t* nerr, int sm_count, cudaStream_t st);
cudaError_t launch_rs_stress_symbols(const RsTables* tab, const uint8_t* gpar, int k, int r, uint64_t seed,
                                     int64_t count, uint8_t* true_cw, uint8_t* recv, int8_t* nerr_true,
                                     cudaStream_t st);
cudaError_t launch_rs_stress(const RsTables* tab, const uint64_t* enc_mask, uint64_t seed, int64_t count,
                             uint64_t* msg, uint64_t* words, int8_t* nerr_true, cudaStream_t st);
cudaError_t launch_swizzle_patterns(const int8_t* pat, int K_pad, int8_t* out, cudaStream_t st);
cudaError_t launch_build_patterns(uint64_t seed, int nbits, int K, int K_pad, int8_t* pat, int32_t* colsum,
                                  cudaStream_t st);
cudaError_t launch_residual(uint64_t seed, int nbits, int K, uint64_t codeword, float* delta, cudaStream_t st);
cudaError_t launch_extract_float(uint64_t seed, int nbits, int K, const float* tile, double* soft, cudaStream_t st);
cudaError_t launch_resample(const GatherDesc& d, int out_w, int out_h, int normalize, void* out, cudaStream_t st);
cudaError_t launch_stage_load(long long ns, cudaStream_t st);
cudaError_t launch_corpus(uint64_t first_seed, int64_t count, int w, int h, int l, int embed, float alpha,
                          const float* delta, uint8_t* out, cudaStream_t st);
}  // namespace qrm

using namespace qrm;

namespace {

// NVTX ranges (tracing): host-side spans of the executor's
// calls, mini-batches and staging, visible in Nsight Systems / ncu; free when
// no tool is attached (NVTX v3 is header-only and dispatches lazily).
struct NvtxRange {
    explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
    ~NvtxRange() { nvtxRangePop(); }
    NvtxRange(const NvtxRange&) = delete;
    NvtxRange& operator=(const NvtxRange&) = delete;
};

}  // namespace

namespace {

// Host CPUs attached to a GPU's NUMA node: /sys/bus/pci/devices/<bus id>/
// local_cpulist (e.g. "0-55,112-167"). Empty when unknown.
std::vector<int> device_cpus(int device) {
    std::vector<int> cpus;
    char bus[32] = {0};
    if (cudaDeviceGetPCIBusId(bus, sizeof bus, device) != cudaSuccess) {
        cudaGetLastError();
        return cpus;
    }
    std::string id(bus);
    for (auto& ch : id) ch = static_cast<char>(std::tolower(static_cast<unsigned char>(ch)));
    std::ifstream f("/sys/bus/pci/devices/" + id + "/local_cpulist");
    std::string list;
    if (!f || !std::getline(f, list)) return cpus;
    size_t pos = 0;
    while (pos < list.size()) {
        size_t end = list.find(',', pos);
        if (end == std::string::npos) end = list.size();
        const std::string part = list.substr(pos, end - pos);
        const size_t dash = part.find('-');
        try {
            const int a = std::stoi(part.substr(0, dash));
            const int b = dash == std::string::npos ? a : std::stoi(part.substr(dash + 1));
            for (int c2 = a; c2 <= b && c2 < CPU_SETSIZE; ++c2) cpus.push_back(c2);
        } catch (...) {
            return {};
        }
        pos = end + 1;
    }
    return cpus;
}

// Pins the calling thread to the GPU's NUMA-local CPUs (no-op when unknown):
// its page-locked buffers are then first-touched on, and read from, that node.
void pin_thread_to_device(int device) {
    const std::vector<int> cpus = device_cpus(device);
    if (cpus.empty()) return;
    cpu_set_t set;
    CPU_ZERO(&set);
    for (int c2 : cpus) CPU_SET(c2, &set);
    pthread_setaffinity_np(pthread_self(), sizeof set, &set);
}

}  // namespace

namespace {

thread_local std::string g_err;
std::atomic<uint64_t> g_launches{0};

qrm_status fail(qrm_status s, const std::string& msg) {
    g_err = msg;
    return s;
}

}  // namespace

// Shared with the other host translation units (formats.cpp).
qrm_status qrm::report_error(qrm_status s, const std::string& msg) { return fail(s, msg); }

namespace {

#define QRM_CUDA(call)                                                                          \
    do {                                                                                        \
        cudaError_t e_ = (call);                                                                \
        if (e_ != cudaSuccess)                                                                  \
            return fail(QRM_CUDA_ERROR, std::string(#call) + ": " + cudaGetErrorString(e_)); \
    } while (0)

#define QRM_LAUNCH(call)       \
    do {                       \
        QRM_CUDA(call);        \
        g_launches.fetch_add(1); \
    } while (0)

cudaStream_t as_stream(void* s) { return reinterpret_cast<cudaStream_t>(s); }

// Runs f when the scope ends, on success and on every early error return.
template <typename F>
struct OnExit {
    F f;
    ~OnExit() { f(); }
};
template <typename F>
OnExit<F> on_exit(F f) {
    return OnExit<F>{f};
}

int64_t now_ns() {
    return std::chrono::duration_cast<std::chrono::nanoseconds>(std::chrono::steady_clock::now().time_since_epoch())
        .count();
}

// Device RS tables per (device, m, n, k), built once.
std::mutex g_tab_mu;
std::map<std::tuple<int, int, int, int>, RsTables*> g_tabs;

qrm_status rs_tables_for(int m, int n, int k, const RsTables** out) {
    int dev = 0;
    QRM_CUDA(cudaGetDevice(&dev));
    std::lock_guard<std::mutex> lock(g_tab_mu);
    auto key = std::make_tuple(dev, m, n, k);
    auto it = g_tabs.find(key);
    if (it != g_tabs.end()) {
        *out = it->second;
        return QRM_OK;
    }
    RsTables h;
    build_rs_tables(m, n, k, h);
    RsTables* d = nullptr;
    QRM_CUDA(cudaMalloc(&d, sizeof(RsTables)));
    QRM_CUDA(cudaMemcpy(d, &h, sizeof(RsTables), cudaMemcpyHostToDevice));
    g_tabs[key] = d;
    *out = d;
    return QRM_OK;
}

template <typename T>
qrm_status ensure(T*& ptr, int64_t& cap, int64_t need) {
    if (need <= cap) return QRM_OK;
    if (ptr) cudaFree(ptr);
    ptr = nullptr;
    cap = 0;
    const int64_t n = std::max<int64_t>(need, 1);
    QRM_CUDA(cudaMalloc(&ptr, sizeof(T) * n));
    cap = n;
    return QRM_OK;
}

struct Workspace {
    int32_t* pending_count = nullptr;
    PendingEntry* pending = nullptr;
    int64_t pending_cap = 0;
    uint8_t* stage = nullptr;  // gathered windows (staged path)
    int64_t stage_cap = 0;
    GatherDesc* descs = nullptr;
    int64_t desc_cap = 0;
    uint8_t* images = nullptr;  // full-image H2D buffer (host pipeline, mode 1)
    int64_t images_cap = 0;
    uint8_t* host_stage = nullptr;  // pinned window staging (host pipeline, mode 2)
    int64_t host_stage_cap = 0;
    void release() {
        if (host_stage) cudaFreeHost(host_stage);
        cudaFree(pending_count);
        cudaFree(pending);
        cudaFree(stage);
        cudaFree(descs);
        cudaFree(images);
        *this = Workspace{};
    }
};

}  // namespace

struct qrm_ctx {
    int device = 0;
    int sms = 148;
    qrm_config cfg{};
    std::vector<uint8_t> key_message;
    int m = 0, n = 0, k = 0, t = 0, nbits = 0, kbits = 0, l = 0, K = 0, K_pad = 0;
    uint64_t key_cw = 0, key_msg = 0;
    int tau_msg = 0, tau_raw = 0;
    int8_t* d_patterns = nullptr;
    int8_t* d_patterns_sw = nullptr;  // per-chunk SW128 smem images of the pattern operand (one bulk copy per stage)
    int32_t* d_colsum = nullptr;
    const RsTables* d_rs = nullptr;
    qrm_record* d_records = nullptr;
    int64_t records_cap = 0;
    std::vector<Workspace> ws;  // [0]: device API; [1..]: host pipeline slots
    std::vector<cudaStream_t> streams;
    qrm_plan plan{{1, 2, 1}, {4096, 4096, 4096}};
    std::unique_ptr<HostPool> pool;  // window staging workers (host pipeline, modes 2 and 3)
    cudaStream_t copy_stream = nullptr;  // mode 3: copy-engine H2D of the staged windows
    std::vector<cudaEvent_t> events;     // host pipeline events, reused call to call
    std::vector<cudaEvent_t> timing_events;  // the same with timing, for calls that report stage spans
    double hybrid_fraction = 0.5;        // mode 3: share of each mini-batch fetched zero-copy
    int64_t stage_piece = 512;           // modes 2/3: windows gathered per H2D
    int64_t stage_grain = 8;             // modes 2/3: windows per host-worker task (sweep: 8 best)
    double decode_ms_per_image = 0.0;  // from the last warm-up profile (Algorithm 2 latencies)
    int extractor = QRM_EXTRACTOR_SPREAD_SPECTRUM;  // qrm_ctx_set_extractor
    bool input_overlap = false;  // qrm_ctx_set_input_overlap
    qrm_record* host_records = nullptr;  // pinned D2H target when the caller's record buffer is pageable
    int64_t host_records_cap = 0;
    // A/B switches, read once at context creation
    int corr_ksplit = 0;            // QRM_CORR_KSPLIT: forced split-K cluster size (0: automatic)
    bool conv_pair = true;          // QRM_CONV_PAIR=0: single-CTA conv layer
    bool conv_fuse_linear = true;   // QRM_CONV_FUSE_LINEAR=0: unfused head
    uint64_t conv_seed = 7;
    // learned (conv) extractor: folded weights + activation ping-pong buffers
    struct Hidden {
        bool ready = false;
        uint64_t seed = 0;
        __nv_bfloat16* w_sw = nullptr;  // [8][9][64][64] swizzled, layers 1..8
        float *bias = nullptr, *w0 = nullptr, *wl = nullptr, *bl = nullptr, *pool = nullptr;
        __nv_bfloat16* act[2] = {nullptr, nullptr};
        int64_t tiles_cap = 0;
        CUtensorMap tmap[2];     // 4-D load maps (conv input)
        CUtensorMap tmap_st[2];  // 2-D store maps (conv output)
    } hid;
};

namespace {

qrm_status workspace_reserve(Workspace& w, int64_t count) {
    qrm_status s;
    if (!w.pending_count) {
        // [0] pending entries, [1] finish-kernel block ticket; re-armed to 0 by
        // the finish kernel itself after every launch.
        QRM_CUDA(cudaMalloc(&w.pending_count, 2 * sizeof(int32_t)));
        QRM_CUDA(cudaMemset(w.pending_count, 0, 2 * sizeof(int32_t)));
    }
    if ((s = ensure(w.pending, w.pending_cap, count)) != QRM_OK) return s;
    return QRM_OK;
}

// Geometry of preprocess (transforms.cpp:24-38).
void geometry(int w, int h, int& up, int& sw, int& sh, int& xo, int& yo) {
    const int mn = std::min(w, h);
    if (mn < kWorkingSize) {
        const double s = static_cast<double>(kWorkingSize) / mn;
        up = 1;
        sw = std::max<int>(kWorkingSize, static_cast<int>(std::lround(w * s)));
        sh = std::max<int>(kWorkingSize, static_cast<int>(std::lround(h * s)));
    } else {
        up = 0;
        sw = w;
        sh = h;
    }
    xo = (sw - kWorkingSize) / 2;
    yo = (sh - kWorkingSize) / 2;
}

DetectParams base_params(qrm_ctx* c, Workspace& w, int64_t count, qrm_record* out, double* soft, uint64_t* raw) {
    DetectParams p{};
    p.count = count;
    p.K = c->K;
    p.K_pad = c->K_pad;
    p.nbits = c->nbits;
    p.kbits = c->kbits;
    p.tau_msg = c->tau_msg;
    p.tau_raw = c->tau_raw;
    p.fuse_t1 = (c->t == 1 && c->n - c->k <= 3) ? 1 : 0;
    p.key_cw = c->key_cw;
    p.key_msg = c->key_msg;
    p.patterns = c->d_patterns;
    p.patterns_sw = c->d_patterns_sw;
    p.colsum = c->d_colsum;
    p.rs = c->d_rs;
    p.out = out;
    p.soft = soft;
    p.raw_out = raw;
    p.pending_count = w.pending_count;
    p.pending = w.pending;
    return p;
}

qrm_status hidden_run(qrm_ctx* c, Workspace& W, const WindowSource& src, int64_t count, qrm_record* out,
                      float* logits, cudaStream_t st);

// Decode + correct `count` windows described by src into device records.
cudaEvent_t g_probe[2] = {nullptr, nullptr};  // set only by qrm_probe_decode_kernel

// wait_inputs: the windows may come from the kernel launched just before on
// `st` (gather, corpus, caller kernels), so the decode must not read them
// before griddepcontrol.wait. Only callers that know the preceding work on `st`
// is complete by stream-event order (the host executor) or is another decode
// (qrm_ctx_set_input_overlap) pass false.
qrm_status run_detect(qrm_ctx* c, Workspace& w, const WindowSource& src, int64_t count, qrm_record* out,
                      double* soft, uint64_t* raw, cudaStream_t st, cudaEvent_t mid_event = nullptr,
                      cudaStream_t finish_stream = nullptr, bool wait_inputs = true, long long load_ns = 0,
                      cudaEvent_t finish_start = nullptr) {
    qrm_status s = workspace_reserve(w, count);
    if (s != QRM_OK) return s;
    if (c->extractor == QRM_EXTRACTOR_CONV) {
        // learned extractor: conv stack + head (+ RS finish) on st
        if ((s = hidden_run(c, w, src, count, out, nullptr, st)) != QRM_OK) return s;
        if (load_ns > 0) QRM_LAUNCH(launch_stage_load(load_ns, st));
        if (mid_event && finish_stream) {
            QRM_CUDA(cudaEventRecord(mid_event, st));
            QRM_CUDA(cudaStreamWaitEvent(finish_stream, mid_event, 0));
            if (finish_start) QRM_CUDA(cudaEventRecord(finish_start, finish_stream));
        }
        return QRM_OK;
    }
    DetectParams p = base_params(c, w, count, out, soft, raw);
    p.src = src;
    if (g_probe[0]) QRM_CUDA(cudaEventRecord(g_probe[0], st));
    p.wait_inputs = wait_inputs ? 1 : 0;
    p.ksplit = c->corr_ksplit;
    QRM_LAUNCH(launch_corr_detect(p, c->sms, st));
    if (g_probe[1]) QRM_CUDA(cudaEventRecord(g_probe[1], st));
    if (load_ns > 0) QRM_LAUNCH(launch_stage_load(load_ns, st));  // SyntheticStageLoad of the decode stage
    cudaStream_t fs = st;
    if (mid_event && finish_stream) {
        QRM_CUDA(cudaEventRecord(mid_event, st));
        QRM_CUDA(cudaStreamWaitEvent(finish_stream, mid_event, 0));
        if (finish_start) QRM_CUDA(cudaEventRecord(finish_start, finish_stream));
        fs = finish_stream;
    }
    // t = 1 codes leave nothing pending (the decode kernel resolves its own ties)
    if (!p.fuse_t1) QRM_LAUNCH(launch_detect_finish(p, std::max(1, c->t), c->sms, fs));
    return QRM_OK;
}

bool direct_ok(const qrm_ctx* c, const uint8_t* base, int w, int h, int64_t stride) {
    int up, sw, sh, xo, yo;
    geometry(w, h, up, sw, sh, xo, yo);
    if (up) return false;
    if (c->cfg.tile_strategy == QRM_TILE_RANDOM) return false;
    const int pitch = w * 3;
    if (reinterpret_cast<uintptr_t>(base) % 16 || stride % 16 || pitch % 16) return false;
    if ((xo * 3) % 16 || (c->l * 3) % 16) return false;
    return true;
}

// Uniform batch at `images` (device-accessible) -> records, choosing the direct
// window path when alignment allows and the gather path otherwise.
// Where the decode kernels read each image's l x l window: straight from the
// images when alignment allows, else from windows staged by the gather kernel.
qrm_status window_source(qrm_ctx* c, Workspace& w, const uint8_t* images, int64_t count, int width, int height,
                         int64_t stride, uint64_t first_draw, cudaStream_t st, WindowSource& src) {
    int up, sw, sh, xo, yo;
    geometry(width, height, up, sw, sh, xo, yo);
    src = WindowSource{};
    src.l = c->l;
    src.strategy = c->cfg.tile_strategy;
    src.tile_seed = c->cfg.tile_seed;
    src.first_draw = first_draw;
    if (direct_ok(c, images, width, height, stride)) {
        src.base = images;
        src.image_stride = stride;
        src.pitch = width * 3;
        src.x_off = xo;
        src.y_off = yo;
        src.direct = 1;
        return QRM_OK;
    }
    qrm_status s;
    if ((s = ensure(w.stage, w.stage_cap, count * c->K)) != QRM_OK) return s;
    if ((s = ensure(w.descs, w.desc_cap, count)) != QRM_OK) return s;
    std::vector<GatherDesc> d(count);
    for (int64_t i = 0; i < count; ++i) {
        int tx, ty;
        select_tile(kWorkingSize, kWorkingSize, c->l, c->cfg.tile_strategy, c->cfg.tile_seed,
                    first_draw + static_cast<uint64_t>(i), tx, ty);
        d[i] = GatherDesc{images + i * stride, width, height, up, sw, sh, xo, yo, tx, ty};
    }
    QRM_CUDA(cudaMemcpyAsync(w.descs, d.data(), sizeof(GatherDesc) * count, cudaMemcpyHostToDevice, st));
    QRM_LAUNCH(launch_gather_windows(w.descs, count, c->l, w.stage, st));
    QRM_CUDA(cudaStreamSynchronize(st));  // the pageable descriptor copy must finish before `d` dies
    src.base = w.stage;
    src.image_stride = c->K;
    src.pitch = 3 * c->l;
    src.direct = 0;
    return QRM_OK;
}

qrm_status detect_uniform(qrm_ctx* c, Workspace& w, const uint8_t* images, int64_t count, int width, int height,
                          int64_t stride, uint64_t first_draw, qrm_record* out, double* soft, uint64_t* raw,
                          cudaStream_t st, cudaEvent_t mid = nullptr, cudaStream_t fs = nullptr,
                          bool overlap_ok = false, long long load_ns = 0, cudaEvent_t finish_start = nullptr) {
    if (count == 0) return QRM_OK;
    WindowSource src;
    const qrm_status s = window_source(c, w, images, count, width, height, stride, first_draw, st, src);
    if (s != QRM_OK) return s;
    // staged windows come from the gather kernel just launched on st
    return run_detect(c, w, src, count, out, soft, raw, st, mid, fs, !(overlap_ok && src.direct), load_ns,
                      finish_start);
}

qrm_status check_uniform(const qrm_ctx* c, const uint8_t* images, int64_t count, int w, int h, int64_t stride) {
    if (!c) return fail(QRM_INVALID_INPUT, "null context");
    if (count < 0) return fail(QRM_INVALID_INPUT, "negative image count");
    if (count > 0 && !images) return fail(QRM_INVALID_INPUT, "null image pointer");
    if (w <= 0 || h <= 0) return fail(QRM_INVALID_INPUT, "image dimensions must be positive");
    if (stride < static_cast<int64_t>(w) * h * 3) return fail(QRM_INVALID_INPUT, "image stride smaller than an image");
    return QRM_OK;
}

qrm_status set_device(int dev) {
    QRM_CUDA(cudaSetDevice(dev));
    return QRM_OK;
}

}  // namespace

extern "C" {

QRM_EXPORT const char* qrm_last_error(void) { return g_err.c_str(); }
QRM_EXPORT int qrm_abi_version(void) { return 1; }
QRM_EXPORT uint64_t qrm_kernel_launch_count(void) { return g_launches.load(); }

QRM_EXPORT int qrm_device_count(void) {
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess) return 0;
    return n;
}

QRM_EXPORT qrm_status qrm_verify_threshold(int n_bits, double fpr, int* tau) {
    const int v = verify_threshold(n_bits, fpr);
    if (v < 0) return fail(QRM_INVALID_INPUT, "verify threshold needs n_bits > 0 and fpr in (0, 1)");
    *tau = v;
    return QRM_OK;
}

QRM_EXPORT qrm_status qrm_rs_encode_packed(int m, int n, int k, uint64_t message, uint64_t* codeword) {
    const std::string e = check_code(m, n, k);
    if (!e.empty()) return fail(QRM_INVALID_INPUT, e);
    if (n * m > 64) return fail(QRM_INVALID_INPUT, "packed words need n*m <= 64");
    *codeword = encode_packed(m, n, k, message);
    return QRM_OK;
}

QRM_EXPORT qrm_status qrm_ctx_create(int device, const qrm_config* cfg, qrm_ctx** out) {
    if (!cfg || !out) return fail(QRM_INVALID_INPUT, "null argument");
    *out = nullptr;
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) return fail(QRM_NO_DEVICE, "no CUDA device available");
    if (device < 0 || device >= ndev) return fail(QRM_INVALID_INPUT, "device index out of range");
    const std::string ce = check_code(cfg->symbol_bits, cfg->n, cfg->k);
    if (!ce.empty()) return fail(QRM_INVALID_INPUT, ce);
    const int nbits = cfg->n * cfg->symbol_bits, kbits = cfg->k * cfg->symbol_bits;
    if (nbits > kMaxNBits) return fail(QRM_INVALID_INPUT, "the detection path supports codewords up to 64 bits");
    if (!cfg->key_message) return fail(QRM_INVALID_INPUT, "key message missing");
    if (cfg->tile_size <= 0 || cfg->tile_size > kWorkingSize) return fail(QRM_INVALID_INPUT, "tile size does not fit image");
    if (cfg->tile_strategy < 0 || cfg->tile_strategy > 2) return fail(QRM_INVALID_INPUT, "unknown tile strategy");
    if (cfg->alpha < 0.0) return fail(QRM_INVALID_INPUT, "alpha must be nonnegative");
    if (!(cfg->fpr_target > 0.0) || !(cfg->fpr_target < 1.0)) return fail(QRM_INVALID_INPUT, "fpr target must be in (0, 1)");
    if ((cfg->n - cfg->k) / 2 > 8) return fail(QRM_INVALID_INPUT, "detection path supports t <= 8");
    qrm_status s = set_device(device);
    if (s != QRM_OK) return s;

    auto c = std::make_unique<qrm_ctx>();
    c->device = device;
    c->cfg = *cfg;
    c->key_message.assign(cfg->key_message, cfg->key_message + kbits);
    c->cfg.key_message = c->key_message.data();
    c->m = cfg->symbol_bits;
    c->n = cfg->n;
    c->k = cfg->k;
    c->t = (cfg->n - cfg->k) / 2;
    c->nbits = nbits;
    c->kbits = kbits;
    c->l = cfg->tile_size;
    c->K = 3 * c->l * c->l;
    c->K_pad = (c->K + 127) / 128 * 128;
    QRM_CUDA(cudaDeviceGetAttribute(&c->sms, cudaDevAttrMultiProcessorCount, device));
    if (const char* e = getenv("QRM_CORR_KSPLIT")) c->corr_ksplit = atoi(e);
    if (const char* e = getenv("QRM_CONV_PAIR")) c->conv_pair = e[0] != '0';
    if (const char* e = getenv("QRM_CONV_FUSE_LINEAR")) c->conv_fuse_linear = e[0] != '0';
    if (const char* e = getenv("QRM_STAGE_PIECE")) c->stage_piece = std::max<int64_t>(16, atoll(e));
    if (const char* e = getenv("QRM_STAGE_GRAIN")) c->stage_grain = std::max<int64_t>(1, atoll(e));
    for (int i = 0; i < kbits; ++i) c->key_msg = (c->key_msg << 1) | (c->key_message[i] & 1);
    c->key_cw = encode_packed(c->m, c->n, c->k, c->key_msg);
    c->tau_msg = verify_threshold(kbits, cfg->fpr_target);
    c->tau_raw = verify_threshold(nbits, cfg->fpr_target);
    if ((s = rs_tables_for(c->m, c->n, c->k, &c->d_rs)) != QRM_OK) return s;
    QRM_CUDA(cudaMalloc(&c->d_patterns, static_cast<size_t>(kMaxNBits) * c->K_pad));
    QRM_CUDA(cudaMalloc(&c->d_colsum, sizeof(int32_t) * kMaxNBits));
    QRM_LAUNCH(launch_build_patterns(cfg->key_seed, nbits, c->K, c->K_pad, c->d_patterns, c->d_colsum, nullptr));
    QRM_CUDA(cudaMalloc(&c->d_patterns_sw, static_cast<size_t>(kMaxNBits) * c->K_pad));
    QRM_LAUNCH(launch_swizzle_patterns(c->d_patterns, c->K_pad, c->d_patterns_sw, nullptr));
    QRM_CUDA(cudaDeviceSynchronize());
    c->ws.resize(1);
    *out = c.release();
    return QRM_OK;
}

QRM_EXPORT void qrm_ctx_destroy(qrm_ctx* c) {
    if (!c) return;
    cudaSetDevice(c->device);
    for (auto& w : c->ws) w.release();
    for (auto s : c->streams) cudaStreamDestroy(s);
    if (c->copy_stream) cudaStreamDestroy(c->copy_stream);
    for (auto e : c->events) cudaEventDestroy(e);
    for (auto e : c->timing_events) cudaEventDestroy(e);
    if (c->host_records) cudaFreeHost(c->host_records);
    cudaFree(c->d_patterns);
    cudaFree(c->d_patterns_sw);
    cudaFree(c->d_colsum);
    cudaFree(c->d_records);
    cudaFree(c->hid.w_sw);
    cudaFree(c->hid.bias);
    cudaFree(c->hid.w0);
    cudaFree(c->hid.wl);
    cudaFree(c->hid.bl);
    cudaFree(c->hid.pool);
    cudaFree(c->hid.act[0]);
    cudaFree(c->hid.act[1]);
    delete c;
}

QRM_EXPORT qrm_status qrm_ctx_info(const qrm_ctx* c, uint64_t* key_codeword, uint64_t* key_message, int* tau_msg,
                                   int* tau_raw) {
    if (!c) return fail(QRM_INVALID_INPUT, "null context");
    if (key_codeword) *key_codeword = c->key_cw;
    if (key_message) *key_message = c->key_msg;
    if (tau_msg) *tau_msg = c->tau_msg;
    if (tau_raw) *tau_raw = c->tau_raw;
    return QRM_OK;
}

QRM_EXPORT qrm_status qrm_ctx_set_plan(qrm_ctx* c, const qrm_plan* plan) {
    if (!c || !plan) return fail(QRM_INVALID_INPUT, "null argument");
    for (int k = 0; k < 3; ++k)
        if (plan->streams[k] < 1 || plan->minibatch[k] < 1) return fail(QRM_INVALID_INPUT, "plan has an empty stage");
    c->plan = *plan;
    return QRM_OK;
}

QRM_EXPORT qrm_status qrm_detect_device(qrm_ctx* c, const uint8_t* images, int64_t count, int w, int h,
                                        int64_t stride, uint64_t first_draw, qrm_record* out, void* stream) {
    NvtxRange range("qrm_detect_device");
    qrm_status s = check_uniform(c, images, count, w, h, stride);
    if (s != QRM_OK) return s;
    if (count > 0 && !out) return fail(QRM_INVALID_INPUT, "null record buffer");
    if ((s = set_device(c->device)) != QRM_OK) return s;
    return detect_uniform(c, c->ws[0], images, count, w, h, stride, first_draw, out, nullptr, nullptr,
                          as_stream(stream), nullptr, nullptr, c->input_overlap);
}

QRM_EXPORT qrm_status qrm_ctx_set_input_overlap(qrm_ctx* c, int enable) {
    if (!c) return fail(QRM_INVALID_INPUT, "null context");
    c->input_overlap = enable != 0;
    return QRM_OK;
}

QRM_EXPORT qrm_status qrm_probe_decode_kernel(qrm_ctx* c, const uint8_t* images, int64_t count, int w, int h,
                                              int64_t stride, int reps, double* avg_ms) {
    qrm_status s = check_uniform(c, images, count, w, h, stride);
    if (s != QRM_OK) return s;
    if (reps < 1 || !avg_ms) return fail(QRM_INVALID_INPUT, "bad probe arguments");
    if ((s = set_device(c->device)) != QRM_OK) return s;
    if ((s = ensure(c->d_records, c->records_cap, count)) != QRM_OK) return s;
    QRM_CUDA(cudaEventCreate(&g_probe[0]));
    QRM_CUDA(cudaEventCreate(&g_probe[1]));
    double total = 0.0;
    for (int i = 0; i < reps && s == QRM_OK; ++i) {
        // a 50 us device spin first, so the decode is already queued when its
        // start event runs: the probe times the launch on the device, not the
        // host's submission latency (~10 us, which an event-to-event span
        // around a lone launch otherwise includes)
        QRM_LAUNCH(launch_stage_load(50000, nullptr));
        s = detect_uniform(c, c->ws[0], images, count, w, h, stride, static_cast<uint64_t>(i) * count, c->d_records,
                           nullptr, nullptr, nullptr, nullptr, nullptr, true);  // resident images, decodes only
        cudaEventSynchronize(g_probe[1]);
        float ms = 0.f;
        cudaEventElapsedTime(&ms, g_probe[0], g_probe[1]);
        total += ms;
    }
    cudaDeviceSynchronize();
    cudaEventDestroy(g_probe[0]);
    cudaEventDestroy(g_probe[1]);
    g_probe[0] = g_probe[1] = nullptr;
    if (s != QRM_OK) return s;
    *avg_ms = total / reps;
    return QRM_OK;
}

QRM_EXPORT qrm_status qrm_extract_device(qrm_ctx* c, const uint8_t* images, int64_t count, int w, int h,
                                         int64_t stride, uint64_t first_draw, double* soft, uint64_t* raw,
                                         void* stream) {
    qrm_status s = check_uniform(c, images, count, w, h, stride);
    if (s != QRM_OK) return s;
    if ((s = set_device(c->device)) != QRM_OK) return s;
    if ((s = ensure(c->d_records, c->records_cap, count)) != QRM_OK) return s;
    return detect_uniform(c, c->ws[0], images, count, w, h, stride, first_draw, c->d_records, soft, raw,
                          as_stream(stream));
}

QRM_EXPORT qrm_status qrm_detect_ragged(qrm_ctx* c, const uint8_t* const* images, const int* widths,
                                        const int* heights, int64_t count, uint64_t first_draw, qrm_record* out) {
    if (!c) return fail(QRM_INVALID_INPUT, "null context");
    if (count < 0) return fail(QRM_INVALID_INPUT, "negative image count");
    if (count == 0) return QRM_OK;
    if (!images || !widths || !heights || !out) return fail(QRM_INVALID_INPUT, "null argument");
    qrm_status s = set_device(c->device);
    if (s != QRM_OK) return s;
    std::vector<int64_t> off(count + 1, 0);
    for (int64_t i = 0; i < count; ++i) {
        if (widths[i] <= 0 || heights[i] <= 0) return fail(QRM_INVALID_INPUT, "image dimensions must be positive");
        if (!images[i]) return fail(QRM_INVALID_INPUT, "null image pointer");
        off[i + 1] = off[i] + static_cast<int64_t>(widths[i]) * heights[i] * 3;
    }
    Workspace& w = c->ws[0];
    if ((s = ensure(w.images, w.images_cap, off[count])) != QRM_OK) return s;
    if ((s = ensure(w.stage, w.stage_cap, count * c->K)) != QRM_OK) return s;
    if ((s = ensure(w.descs, w.desc_cap, count)) != QRM_OK) return s;
    if ((s = ensure(c->d_records, c->records_cap, count)) != QRM_OK) return s;
    for (int64_t i = 0; i < count; ++i)
        QRM_CUDA(cudaMemcpy(w.images + off[i], images[i], off[i + 1] - off[i], cudaMemcpyHostToDevice));
    std::vector<GatherDesc> d(count);
    for (int64_t i = 0; i < count; ++i) {
        int up, sw, sh, xo, yo, tx, ty;
        geometry(widths[i], heights[i], up, sw, sh, xo, yo);
        select_tile(kWorkingSize, kWorkingSize, c->l, c->cfg.tile_strategy, c->cfg.tile_seed,
                    first_draw + static_cast<uint64_t>(i), tx, ty);
        d[i] = GatherDesc{w.images + off[i], widths[i], heights[i], up, sw, sh, xo, yo, tx, ty};
    }
    QRM_CUDA(cudaMemcpy(w.descs, d.data(), sizeof(GatherDesc) * count, cudaMemcpyHostToDevice));
    QRM_LAUNCH(launch_gather_windows(w.descs, count, c->l, w.stage, nullptr));
    WindowSource src{};
    src.base = w.stage;
    src.image_stride = c->K;
    src.pitch = 3 * c->l;
    src.direct = 0;
    src.l = c->l;
    src.strategy = c->cfg.tile_strategy;
    src.tile_seed = c->cfg.tile_seed;
    src.first_draw = first_draw;
    if ((s = run_detect(c, w, src, count, c->d_records, nullptr, nullptr, nullptr)) != QRM_OK) return s;
    QRM_CUDA(cudaMemcpy(out, c->d_records, sizeof(qrm_record) * count, cudaMemcpyDeviceToHost));
    return QRM_OK;
}

}  // extern "C"

namespace {

qrm_status tensor_map_encoder(PFN_cuTensorMapEncodeTiled_v12000* out);

// 3-D TMA view of `count` uniform u8 images ([count][h][3w], any image stride):
// box = one 64-row x 192-B window (tile_bf16_kernel, fetch_windows_tma_kernel).
qrm_status encode_window_map(CUtensorMap* map, const uint8_t* base, int w, int h, int64_t stride, int64_t count) {
    PFN_cuTensorMapEncodeTiled_v12000 encode = nullptr;
    qrm_status s = tensor_map_encoder(&encode);
    if (s != QRM_OK) return s;
    const cuuint64_t dims[3] = {static_cast<cuuint64_t>(w) * 3, static_cast<cuuint64_t>(h), static_cast<cuuint64_t>(count)};
    const cuuint64_t strides[2] = {static_cast<cuuint64_t>(w) * 3, static_cast<cuuint64_t>(stride)};
    const cuuint32_t box[3] = {192, 64, 1};
    const cuuint32_t estr[3] = {1, 1, 1};
    const CUresult r = encode(map, CU_TENSOR_MAP_DATA_TYPE_UINT8, 3, const_cast<uint8_t*>(base), dims, strides, box, estr,
                              CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_64B,
                              CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) return fail(QRM_CUDA_ERROR, "cuTensorMapEncodeTiled (windows) failed (" + std::to_string(r) + ")");
    return QRM_OK;
}

// Transfer stage of host-pipeline modes 0/3: `count` windows described by the
// direct source `hs` (mapped host images) -> contiguous device windows. 64x64
// tiles: one TMA box per window (fetch_windows_tma_kernel, 3.74 vs 3.64 M
// img/s end to end); other sizes: 16-B zero-copy loads (fetch_windows_kernel).
qrm_status fetch_stage(const qrm_ctx* c, const WindowSource& hs, int w, int h, int64_t count, uint8_t* dst,
                       cudaStream_t st) {
    if (count <= 0) return QRM_OK;
    if (c->l == 64) {
        CUtensorMap fm;
        qrm_status s = encode_window_map(&fm, hs.base, w, h, hs.image_stride, count);
        if (s != QRM_OK) return s;
        QRM_LAUNCH(launch_fetch_windows_tma(fm, hs, count, dst, c->sms, st));
    } else {
        QRM_LAUNCH(launch_fetch_windows(hs, count, c->K, dst, c->sms, st));
    }
    return QRM_OK;
}

// One unit of work of the host executor: images [first, first + count) decoded
// on decode stream `stream` (its workspace slot). Round-robin mini-batches, or
// the pieces of an Algorithm-2 schedule.
struct HostPiece {
    int64_t first, count;
    int stream;
};

// Optional parts of a host-pipeline call.
struct HostCallOpts {
    const uint8_t* const* ptrs = nullptr;  // per-image host addresses (qrm_detect_host_images): staged transfer
    const qrm_stage_load* load = nullptr;  // SyntheticStageLoad
    qrm_stage_times* times = nullptr;      // DeskReport / StageLatencies accounting
};

qrm_status detect_host_impl(qrm_ctx* c, const uint8_t* images, int64_t count, int w, int h, int64_t stride,
                            uint64_t first_draw, qrm_record* out, const qrm_plan* plan, int mode,
                            qrm_host_stats* stats, const std::vector<HostPiece>* pieces,
                            const HostCallOpts& opt = HostCallOpts{}) {
    NvtxRange call_range("qrm_detect_host");
    qrm_status s;
    if (opt.ptrs) {
        if (!c) return fail(QRM_INVALID_INPUT, "null context");
        if (count < 0) return fail(QRM_INVALID_INPUT, "negative image count");
        if (w <= 0 || h <= 0) return fail(QRM_INVALID_INPUT, "image dimensions must be positive");
        for (int64_t i = 0; i < count; ++i)
            if (!opt.ptrs[i]) return fail(QRM_INVALID_INPUT, "null image pointer");
        mode = 2;  // separate pageable images: only their windows are staged and copied
    } else if ((s = check_uniform(c, images, count, w, h, stride)) != QRM_OK) {
        return s;
    }
    if (count > 0 && !out) return fail(QRM_INVALID_INPUT, "null record buffer");
    if (mode < 0 || mode > 3)
        return fail(QRM_INVALID_INPUT,
                    "mode must be 0 (mapped window), 1 (full image), 2 (staged window) or 3 (mapped + staged)");
    if ((s = set_device(c->device)) != QRM_OK) return s;
    const qrm_plan P = plan ? *plan : c->plan;
    for (int k = 0; k < 3; ++k)
        if (P.streams[k] < 1 || P.minibatch[k] < 1) return fail(QRM_INVALID_INPUT, "plan has an empty stage");
    long long load_ns[3] = {0, 0, 0};
    if (opt.load)
        for (int k = 0; k < 3; ++k) {
            if (opt.load->ns[k] < 0) return fail(QRM_INVALID_INPUT, "synthetic stage load must be >= 0");
            load_ns[k] = opt.load->ns[k];
        }
    const int64_t t0 = now_ns();
    if (opt.times) {
        opt.times->wall_ns = 0;
        for (int k = 0; k < 3; ++k) opt.times->busy_ns[k] = 0;
    }
    if (count == 0) return QRM_OK;
    const int64_t img_bytes = static_cast<int64_t>(w) * h * 3;
    int up, sw, sh, xo, yo;
    geometry(w, h, up, sw, sh, xo, yo);
    if (opt.ptrs && up) return fail(QRM_INVALID_INPUT, "per-image host batches need min(w, h) >= 256 (use the ragged path)");
    auto image_at = [&](int64_t i) -> const uint8_t* { return opt.ptrs ? opt.ptrs[i] : images + i * stride; };

    // Host buffers must be page-locked and mapped; register them for the call if not.
    const int64_t in_bytes = opt.ptrs ? 0 : (count - 1) * stride + img_bytes;
    bool reg_in = false, reg_out = false;
    int nstreams_used = 0;
    // Every exit path (errors included) drains the streams this call used
    // before the context's events are reused and the caller's buffers unregistered.
    auto cleanup = on_exit([&] {
        for (int i = 0; i < nstreams_used; ++i) cudaStreamSynchronize(c->streams[i]);
        if (c->copy_stream) cudaStreamSynchronize(c->copy_stream);
        if (reg_in) cudaHostUnregister(const_cast<uint8_t*>(images));
        if (reg_out) cudaHostUnregister(out);
    });
    cudaPointerAttributes attr{};
    uint8_t* dimg = nullptr;
    if (!opt.ptrs) {
        if (cudaPointerGetAttributes(&attr, images) != cudaSuccess || attr.type != cudaMemoryTypeHost) {
            cudaGetLastError();
            QRM_CUDA(cudaHostRegister(const_cast<uint8_t*>(images), in_bytes,
                                      cudaHostRegisterMapped | cudaHostRegisterReadOnly));
            reg_in = true;
        }
        QRM_CUDA(cudaHostGetDevicePointer(reinterpret_cast<void**>(&dimg), const_cast<uint8_t*>(images), 0));
    }
    // Records go D2H into pinned memory: the caller's buffer when it is pinned,
    // else the context's pinned record buffer (copied out at the end; cheaper
    // than registering the caller's buffer every call).
    qrm_record* hout = out;
    if (cudaPointerGetAttributes(&attr, out) != cudaSuccess || attr.type != cudaMemoryTypeHost) {
        cudaGetLastError();
        if (c->host_records_cap < count) {
            if (c->host_records) cudaFreeHost(c->host_records);
            c->host_records = nullptr;
            c->host_records_cap = 0;
            QRM_CUDA(cudaHostAlloc(&c->host_records, sizeof(qrm_record) * count, cudaHostAllocDefault));
            c->host_records_cap = count;
        }
        hout = c->host_records;
    }

    // Streams: [0, s0) transfer, [s0, s0+s1) decode, [s0+s1, s0+s1+s2) correct/return.
    const int s0 = P.streams[0], s1 = P.streams[1], s2 = P.streams[2];
    const int nstreams = s0 + s1 + s2;
    while (static_cast<int>(c->streams.size()) < nstreams) {
        cudaStream_t st;
        QRM_CUDA(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
        c->streams.push_back(st);
    }
    const int64_t mb = P.minibatch[1];
    const int64_t nmb = (count + mb - 1) / mb;
    // One workspace per decode stream slot (pending lists are per launch).
    if (static_cast<int>(c->ws.size()) < 1 + s1) c->ws.resize(1 + s1);
    if ((s = ensure(c->d_records, c->records_cap, count)) != QRM_OK) return s;
    // Full-image mode: one device image buffer per decode slot.
    if ((mode == 2 || mode == 3) && up) mode = 1;  // upscaled inputs need the device bilinear gather
    if (mode == 3 && !(direct_ok(c, dimg, w, h, stride) && (3 * c->l) % 16 == 0)) mode = 2;
    if (mode == 1)
        for (int j = 0; j < s1; ++j)
            if ((s = ensure(c->ws[1 + j].images, c->ws[1 + j].images_cap, mb * img_bytes)) != QRM_OK) return s;
    if (mode == 2 || mode == 3) {
        if (mode == 3 && !c->copy_stream) QRM_CUDA(cudaStreamCreateWithFlags(&c->copy_stream, cudaStreamNonBlocking));
        if (!c->pool) {
            const unsigned hc = std::thread::hardware_concurrency();
            const int dev = c->device;
            c->pool = std::make_unique<HostPool>(static_cast<int>(std::max(1u, std::min(hc ? hc - 1 : 1u, 31u))),
                                                 [dev] { pin_thread_to_device(dev); });
        }
        for (int j = 0; j < s1; ++j) {
            Workspace& W = c->ws[1 + j];
            if ((s = ensure(W.stage, W.stage_cap, mb * c->K)) != QRM_OK) return s;
            if (W.host_stage_cap < mb * c->K) {  // the context's pinned staging ring, reused call to call
                if (W.host_stage) cudaFreeHost(W.host_stage);
                W.host_stage = nullptr;
                W.host_stage_cap = 0;
                QRM_CUDA(cudaHostAlloc(&W.host_stage, mb * c->K, cudaHostAllocDefault));
                W.host_stage_cap = mb * c->K;
            }
        }
    }

    // One mini-batch, zero-copy transfer: the whole call on one stream. The
    // decode launches behind the window fetch (programmatic dependent launch,
    // its producers wait for the fetch) and writes the records straight into
    // the page-locked host buffer, so there are no cross-stream event hops and
    // no D2H copy: ~50 -> ~35 us of fixed cost per call.
    if (!pieces && nmb == 1 && mode == 0 && !opt.ptrs && !opt.times && load_ns[0] == 0 && load_ns[1] == 0 &&
        load_ns[2] == 0 && !up && dimg && c->extractor == QRM_EXTRACTOR_SPREAD_SPECTRUM &&
        direct_ok(c, dimg, w, h, stride) && (3 * c->l) % 16 == 0) {
        qrm_record* dout = nullptr;
        if (cudaHostGetDevicePointer(reinterpret_cast<void**>(&dout), hout, 0) == cudaSuccess && dout) {
            cudaStream_t st = c->streams[0];
            nstreams_used = 1;
            Workspace& W = c->ws[1];
            if ((s = ensure(W.stage, W.stage_cap, count * c->K)) != QRM_OK) return s;
            const int launches0 = static_cast<int>(g_launches.load());
            WindowSource hs{};
            hs.base = dimg;
            hs.image_stride = stride;
            hs.pitch = w * 3;
            hs.x_off = xo;
            hs.y_off = yo;
            hs.direct = 1;
            hs.l = c->l;
            hs.strategy = c->cfg.tile_strategy;
            hs.tile_seed = c->cfg.tile_seed;
            hs.first_draw = first_draw;
            if ((s = fetch_stage(c, hs, w, h, count, W.stage, st)) != QRM_OK) return s;
            WindowSource ws = hs;
            ws.base = W.stage;
            ws.image_stride = c->K;
            ws.pitch = 3 * c->l;
            ws.direct = 0;
            if ((s = run_detect(c, W, ws, count, dout, nullptr, nullptr, st, nullptr, nullptr, true)) != QRM_OK)
                return s;
            QRM_CUDA(cudaStreamSynchronize(st));
            if (hout != out) std::memcpy(out, hout, sizeof(qrm_record) * count);
            if (stats) {
                stats->wall_ms = static_cast<double>(now_ns() - t0) / 1e6;
                stats->h2d_bytes = static_cast<double>(c->K) * count;
                stats->d2h_bytes = static_cast<double>(sizeof(qrm_record)) * count;
                stats->minibatches = 1;
                stats->kernel_launches = static_cast<int>(g_launches.load()) - launches0;
            }
            return QRM_OK;
        }
        cudaGetLastError();
    }

    nstreams_used = nstreams;
    const int64_t nwork = pieces ? static_cast<int64_t>(pieces->size()) : nmb;
    // events come from the context's pools (creating ~20 per call cost ~50 us);
    // timing-enabled ones only when the call asks for stage accounting
    const bool timed = opt.times != nullptr;
    std::vector<cudaEvent_t>& pool_ev = timed ? c->timing_events : c->events;
    const size_t nev = static_cast<size_t>(4 * nstreams + 8 * nwork);
    while (pool_ev.size() < nev) {
        cudaEvent_t e;
        QRM_CUDA(cudaEventCreateWithFlags(&e, timed ? cudaEventDefault : cudaEventDisableTiming));
        pool_ev.push_back(e);
    }
    const std::vector<cudaEvent_t>& ev = pool_ev;
    size_t evi = 0;
    // per work item: stage k spans [span[b][2k], span[b][2k+1]] (timed calls)
    std::vector<std::array<cudaEvent_t, 6>> span(timed ? nwork : 0);
    std::vector<cudaEvent_t> slot_free(s1, nullptr);  // decode slot j reusable after its last finish
    double h2d = 0.0;
    int launches0 = static_cast<int>(g_launches.load());
    for (int64_t b = 0; b < nwork; ++b) {
        NvtxRange mb_range("mini-batch");
        const int64_t first = pieces ? (*pieces)[b].first : b * mb;
        const int64_t cnt = pieces ? (*pieces)[b].count : std::min(mb, count - first);
        const int lane = pieces ? (*pieces)[b].stream : static_cast<int>(b % s1);
        cudaStream_t xs = c->streams[b % s0];
        // the conv extractor's activation buffers are per context: one decode stream
        cudaStream_t ds = c->streams[s0 + (c->extractor == QRM_EXTRACTOR_CONV ? 0 : lane)];
        cudaStream_t cs = c->streams[s0 + s1 + b % s2];
        const int slot = lane;
        Workspace& W = c->ws[1 + slot];
        const uint8_t* src = dimg ? dimg + first * stride : nullptr;
        int64_t src_stride = stride;
        cudaEvent_t e_in = ev[evi++], e_mid = ev[evi++], e_done = ev[evi++];
        cudaEvent_t t0s = nullptr, t1s = nullptr, t2s = nullptr;
        if (timed) {
            t0s = ev[evi++];
            t1s = ev[evi++];
            t2s = ev[evi++];
            span[b] = {t0s, e_in, t1s, e_mid, t2s, e_done};
        }
        if (slot_free[slot]) QRM_CUDA(cudaStreamWaitEvent(xs, slot_free[slot], 0));
        if (t0s) QRM_CUDA(cudaEventRecord(t0s, xs));
        const long long ld0 = load_ns[0] * cnt, ld1 = load_ns[1] * cnt, ld2 = load_ns[2] * cnt;
        // stage 1 (decode) on ds once stage 0 is done, stage 2 (complete + return) on cs
        auto start_decode = [&]() -> qrm_status {
            QRM_CUDA(cudaStreamWaitEvent(ds, e_in, 0));
            if (t1s) QRM_CUDA(cudaEventRecord(t1s, ds));
            return QRM_OK;
        };
        auto finish_return = [&]() -> qrm_status {
            QRM_CUDA(cudaMemcpyAsync(hout + first, c->d_records + first, sizeof(qrm_record) * cnt,
                                     cudaMemcpyDeviceToHost, cs));
            if (ld2 > 0) QRM_LAUNCH(launch_stage_load(ld2, cs));
            QRM_CUDA(cudaEventRecord(e_done, cs));
            slot_free[slot] = e_done;
            return QRM_OK;
        };
        if (mode == 2 || mode == 3) {
            // stage 0. Mode 3: the transfer kernel pulls the first `nz` windows
            // over PCIe (zero-copy) while the CPU workers copy the others into
            // pinned staging for one copy-engine H2D on the copy stream; the two
            // share the link (round-1 PCIe probe: 47.8 GB/s zero-copy alone,
            // 50.9 GB/s half and half). Mode 2: all windows through staging.
            const int K = c->K;
            const int64_t nz = mode == 3 ? std::min(cnt, static_cast<int64_t>(c->hybrid_fraction * cnt)) : 0;
            WindowSource hs{};
            hs.base = src;
            hs.image_stride = stride;
            hs.pitch = w * 3;
            hs.x_off = xo;
            hs.y_off = yo;
            hs.direct = 1;
            hs.l = c->l;
            hs.strategy = c->cfg.tile_strategy;
            hs.tile_seed = c->cfg.tile_seed;
            hs.first_draw = first_draw + static_cast<uint64_t>(first);
            if (nz > 0 && (s = fetch_stage(c, hs, w, h, nz, W.stage, xs)) != QRM_OK) return s;
            if (slot_free[slot]) QRM_CUDA(cudaEventSynchronize(slot_free[slot]));  // host_stage reusable
            uint8_t* hst = W.host_stage;
            const int l = c->l, rowb = 3 * l, pitch = 3 * w;
            const auto& cfg = c->cfg;
            cudaStream_t cps = mode == 3 ? c->copy_stream : xs;
            if (mode == 3 && slot_free[slot]) QRM_CUDA(cudaStreamWaitEvent(cps, slot_free[slot], 0));
            // the staged windows in pieces: the copy engine moves piece j while
            // the workers gather piece j + 1
            const int64_t piece = c->stage_piece;
            for (int64_t p0 = 0; p0 < cnt - nz; p0 += piece) {
                const int64_t p1 = std::min(cnt - nz, p0 + piece);
                NvtxRange gather_range("stage windows (host gather)");
                c->pool->parallel_for(p1 - p0, c->stage_grain, [&](int64_t j0, int64_t j1) {
                    auto window_at = [&](int64_t i) {
                        const int64_t img = first + nz + i;
                        int tx, ty;
                        select_tile(kWorkingSize, kWorkingSize, l, cfg.tile_strategy, cfg.tile_seed,
                                    first_draw + static_cast<uint64_t>(img), tx, ty);
                        return image_at(img) + static_cast<int64_t>(yo + ty) * pitch + static_cast<int64_t>(xo + tx) * 3;
                    };
                    // The windows' rows are cold (each image is read once): prefetch the
                    // next window's 64 rows while this one is copied, so the worker has a
                    // whole window of line fills in flight instead of one row's.
                    const uint8_t* next = j0 < j1 ? window_at(p0 + j0) : nullptr;
                    for (int64_t i = p0 + j0; i < p0 + j1; ++i) {
                        const uint8_t* src0 = next;
                        next = i + 1 < p0 + j1 ? window_at(i + 1) : nullptr;
                        if (next && rowb == 192)
                            for (int r = 0; r < 64; ++r) {
                                const char* row = reinterpret_cast<const char*>(next + static_cast<int64_t>(r) * pitch);
                                _mm_prefetch(row, _MM_HINT_T0);
                                _mm_prefetch(row + 64, _MM_HINT_T0);
                                _mm_prefetch(row + 128, _MM_HINT_T0);
                                _mm_prefetch(row + 191, _MM_HINT_T0);
                            }
                        uint8_t* dst = hst + i * K;
                        if (rowb == 192) {
                            // l = 64: non-temporal 16-B stores. Staging written through
                            // the cache stays dirty in the workers' L2s and the copy
                            // engine's reads of it crawl (50 MB: 3.0 ms vs 0.92 ms)
                            for (int r = 0; r < 64; ++r) {
                                const __m128i* s16 = reinterpret_cast<const __m128i*>(src0 + static_cast<int64_t>(r) * pitch);
                                __m128i* d16 = reinterpret_cast<__m128i*>(dst + r * 192);
                                for (int k = 0; k < 12; ++k) _mm_stream_si128(d16 + k, _mm_loadu_si128(s16 + k));
                            }
                        } else
                            for (int r = 0; r < l; ++r)
                                std::memcpy(dst + r * rowb, src0 + static_cast<int64_t>(r) * pitch, rowb);
                    }
                    _mm_sfence();  // the streaming stores are globally visible before the H2D is issued
                });
                QRM_CUDA(cudaMemcpyAsync(W.stage + (nz + p0) * K, hst + p0 * K, (p1 - p0) * K, cudaMemcpyHostToDevice,
                                         cps));
            }
            h2d += static_cast<double>(K) * cnt;
            if (ld0 > 0) QRM_LAUNCH(launch_stage_load(ld0, xs));
            QRM_CUDA(cudaEventRecord(e_in, xs));
            if (mode == 3) {  // the staged share arrives on the copy stream
                cudaEvent_t e_cp = ev[evi++];
                QRM_CUDA(cudaEventRecord(e_cp, cps));
                QRM_CUDA(cudaStreamWaitEvent(ds, e_cp, 0));
            }
            if ((s = start_decode()) != QRM_OK) return s;
            WindowSource ws = hs;
            ws.base = W.stage;
            ws.image_stride = K;
            ws.pitch = rowb;
            ws.direct = 0;
            ws.x_off = 0;
            ws.y_off = 0;
            // the windows are complete by event order (e_in); only a decode precedes on ds
            if ((s = run_detect(c, W, ws, cnt, c->d_records + first, nullptr, nullptr, ds, e_mid, cs, false, ld1,
                                t2s)) != QRM_OK)
                return s;
            if ((s = finish_return()) != QRM_OK) return s;
            continue;
        }
        if (mode == 0 && direct_ok(c, src, w, h, stride) && (3 * c->l) % 16 == 0) {
            // stage 0: the transfer kernel pulls each window over PCIe (zero-copy
            // reads of mapped host memory) into this slot's device windows
            if ((s = ensure(W.stage, W.stage_cap, mb * c->K)) != QRM_OK) return s;
            WindowSource hs{};
            hs.base = src;
            hs.image_stride = stride;
            hs.pitch = w * 3;
            hs.x_off = xo;
            hs.y_off = yo;
            hs.direct = 1;
            hs.l = c->l;
            hs.strategy = c->cfg.tile_strategy;
            hs.tile_seed = c->cfg.tile_seed;
            hs.first_draw = first_draw + static_cast<uint64_t>(first);
            if ((s = fetch_stage(c, hs, w, h, cnt, W.stage, xs)) != QRM_OK) return s;
            h2d += static_cast<double>(c->K) * cnt;
            if (ld0 > 0) QRM_LAUNCH(launch_stage_load(ld0, xs));
            QRM_CUDA(cudaEventRecord(e_in, xs));
            if ((s = start_decode()) != QRM_OK) return s;
            WindowSource ws = hs;
            ws.base = W.stage;
            ws.image_stride = c->K;
            ws.pitch = 3 * c->l;
            ws.direct = 0;
            // the windows are complete by event order (e_in); only a decode precedes on ds
            if ((s = run_detect(c, W, ws, cnt, c->d_records + first, nullptr, nullptr, ds, e_mid, cs, false, ld1,
                                t2s)) != QRM_OK)
                return s;
            if ((s = finish_return()) != QRM_OK) return s;
            continue;
        }
        if (mode == 1) {
            // stage 0: H2D of the mini-batch's full images on the copy stream
            QRM_CUDA(cudaMemcpy2DAsync(W.images, img_bytes, images + first * stride, stride, img_bytes, cnt,
                                       cudaMemcpyHostToDevice, xs));
            h2d += static_cast<double>(img_bytes) * cnt;
            src = W.images;
            src_stride = img_bytes;
        } else {
            h2d += static_cast<double>(c->K) * cnt;  // window bytes read over PCIe by the decode kernel
        }
        if (ld0 > 0) QRM_LAUNCH(launch_stage_load(ld0, xs));
        QRM_CUDA(cudaEventRecord(e_in, xs));
        if (slot_free[slot]) QRM_CUDA(cudaStreamWaitEvent(ds, slot_free[slot], 0));
        if ((s = start_decode()) != QRM_OK) return s;
        if ((s = detect_uniform(c, W, src, cnt, w, h, src_stride, first_draw + static_cast<uint64_t>(first),
                                c->d_records + first, nullptr, nullptr, ds, e_mid, cs, true, ld1, t2s)) != QRM_OK)
            return s;
        if ((s = finish_return()) != QRM_OK) return s;
    }
    for (int i = 0; i < nstreams; ++i) QRM_CUDA(cudaStreamSynchronize(c->streams[i]));
    if (c->copy_stream) QRM_CUDA(cudaStreamSynchronize(c->copy_stream));
    if (hout != out) std::memcpy(out, hout, sizeof(qrm_record) * count);
    if (stats) {
        stats->wall_ms = static_cast<double>(now_ns() - t0) / 1e6;
        stats->h2d_bytes = h2d;
        stats->d2h_bytes = static_cast<double>(sizeof(qrm_record)) * count;
        stats->minibatches = static_cast<int>(nmb);
        stats->kernel_launches = static_cast<int>(g_launches.load()) - launches0;
    }
    if (timed) {
        for (int64_t b = 0; b < nwork; ++b) {
            const int64_t first = pieces ? (*pieces)[b].first : b * mb;
            const int64_t cnt = pieces ? (*pieces)[b].count : std::min(mb, count - first);
            for (int k = 0; k < 3; ++k) {
                float ms = 0.f;
                QRM_CUDA(cudaEventElapsedTime(&ms, span[b][2 * k], span[b][2 * k + 1]));
                const int64_t ns = static_cast<int64_t>(static_cast<double>(ms) * 1e6);
                opt.times->busy_ns[k] += ns;
                if (opt.times->image_ns)
                    for (int64_t i = first; i < first + cnt; ++i) opt.times->image_ns[3 * i + k] = ns;
            }
        }
        opt.times->wall_ns = now_ns() - t0;
    }
    return QRM_OK;
}

}  // namespace

extern "C" {

QRM_EXPORT qrm_status qrm_detect_host(qrm_ctx* c, const uint8_t* images, int64_t count, int w, int h,
                                      int64_t stride, uint64_t first_draw, qrm_record* out, const qrm_plan* plan,
                                      int mode, qrm_host_stats* stats) {
    return detect_host_impl(c, images, count, w, h, stride, first_draw, out, plan, mode, stats, nullptr);
}

QRM_EXPORT qrm_status qrm_detect_host_timed(qrm_ctx* c, const uint8_t* images, int64_t count, int w, int h,
                                            int64_t stride, uint64_t first_draw, qrm_record* out, const qrm_plan* plan,
                                            int mode, const qrm_stage_load* load, qrm_stage_times* times) {
    HostCallOpts o;
    o.load = load;
    o.times = times;
    return detect_host_impl(c, images, count, w, h, stride, first_draw, out, plan, mode, nullptr, nullptr, o);
}

QRM_EXPORT qrm_status qrm_detect_host_images(qrm_ctx* c, const uint8_t* const* images, int64_t count, int w, int h,
                                             uint64_t first_draw, qrm_record* out, const qrm_plan* plan,
                                             const qrm_stage_load* load, qrm_stage_times* times) {
    if (count > 0 && !images) return fail(QRM_INVALID_INPUT, "null image pointer array");
    HostCallOpts o;
    o.ptrs = images;
    o.load = load;
    o.times = times;
    return detect_host_impl(c, nullptr, count, w, h, static_cast<int64_t>(w) * h * 3, first_draw, out, plan, 2,
                            nullptr, nullptr, o);
}

QRM_EXPORT qrm_status qrm_detect_host_lpt(qrm_ctx* c, const uint8_t* images, int64_t count, int w, int h,
                                          int64_t stride, uint64_t first_draw, qrm_record* out, const qrm_plan* plan,
                                          int mode, double lambda, int b_min, qrm_host_stats* stats) {
    // Resource-aware mini-batch scheduling (section 6.2, Algorithm 2;
    // lpt_schedule, sched.cpp:177-235) driving the executor: tasks are the
    // mini-batches of plan.minibatch[1] images, their latency the decode stage's
    // per-image time from this context's warm-up profile (uniform when none was
    // taken) and their memory the staged-window bytes; LPT places them on the
    // plan.streams[1] decode streams, sharding into b_min-image pieces where
    // the balance slack lambda demands. Each piece runs on its assigned stream.
    qrm_status s = check_uniform(c, images, count, w, h, stride);
    if (s != QRM_OK) return s;
    const qrm_plan P = plan ? *plan : c->plan;
    if (P.streams[1] < 1 || P.minibatch[1] < 1) return fail(QRM_INVALID_INPUT, "plan has an empty stage");
    if (b_min < 1) return fail(QRM_INVALID_INPUT, "b_min must be >= 1");
    if (count == 0) return detect_host_impl(c, images, 0, w, h, stride, first_draw, out, plan, mode, stats, nullptr);
    const int64_t mb = P.minibatch[1];
    const int64_t nmb = (count + mb - 1) / mb;
    if (nmb > INT32_MAX) return fail(QRM_INVALID_INPUT, "too many mini-batches");
    const double per_image = c->decode_ms_per_image > 0.0 ? c->decode_ms_per_image : 1.0;
    std::vector<sched::Task> tasks(static_cast<size_t>(nmb));
    for (int64_t t = 0; t < nmb; ++t) {
        const int64_t cnt = std::min(mb, count - t * mb);
        tasks[t].id = static_cast<int>(t);
        tasks[t].units = static_cast<int>(cnt);
        tasks[t].latency = per_image * static_cast<double>(cnt);
        tasks[t].memory = static_cast<double>(c->K) * static_cast<double>(cnt);
    }
    size_t free_b = 0, total_b = 0;
    if ((s = set_device(c->device)) != QRM_OK) return s;
    QRM_CUDA(cudaMemGetInfo(&free_b, &total_b));
    sched::Schedule sch;
    std::string err;
    const int rc = sched::lpt_schedule(tasks, P.streams[1], lambda, static_cast<double>(free_b), b_min,
                                       static_cast<int>(std::min<int64_t>(count, INT32_MAX)), sch, err);
    if (rc) return fail(static_cast<qrm_status>(rc), err);
    // pieces of a task are consecutive image ranges in placement order
    std::vector<int64_t> offset(static_cast<size_t>(nmb), 0);
    std::vector<HostPiece> pieces;
    for (int st = 0; st < P.streams[1]; ++st)
        for (const auto& t : sch.streams[st]) {
            const int64_t first = static_cast<int64_t>(t.id) * mb + offset[t.id];
            pieces.push_back(HostPiece{first, t.units, st});
            offset[t.id] += t.units;
        }
    int64_t covered = 0;
    for (int64_t t = 0; t < nmb; ++t) covered += offset[t];
    if (covered != count) return fail(QRM_INFEASIBLE, "schedule does not cover the batch");
    // issue in placement order, interleaving the streams (piece i of every stream, then i+1, ...)
    std::vector<HostPiece> order;
    std::vector<size_t> next(P.streams[1], 0);
    std::vector<std::vector<HostPiece>> per(P.streams[1]);
    for (const auto& pc : pieces) per[pc.stream].push_back(pc);
    for (bool more = true; more;) {
        more = false;
        for (int st = 0; st < P.streams[1]; ++st)
            if (next[st] < per[st].size()) {
                order.push_back(per[st][next[st]++]);
                more = true;
            }
    }
    return detect_host_impl(c, images, count, w, h, stride, first_draw, out, plan, mode, stats, &order);
}

QRM_EXPORT qrm_status qrm_detect_host_multi(qrm_ctx* const* ctxs, int nctx, const uint8_t* images, int64_t count,
                                            int w, int h, int64_t stride, uint64_t first_draw, qrm_record* out,
                                            const qrm_plan* plan, int mode, qrm_host_stats* stats) {
    // detect_batch over several devices of one node: images are
    // independent, so context i takes the contiguous shard
    // [count*i/n, count*(i+1)/n) with its GLOBAL draw indices, on its own host
    // thread; records land at their global positions. No collective.
    if (!ctxs || nctx < 1) return fail(QRM_INVALID_INPUT, "need at least one context");
    for (int i = 0; i < nctx; ++i)
        if (!ctxs[i]) return fail(QRM_INVALID_INPUT, "null context");
    qrm_status s = check_uniform(ctxs[0], images, count, w, h, stride);
    if (s != QRM_OK) return s;
    if (count > 0 && !out) return fail(QRM_INVALID_INPUT, "null record buffer");
    const int64_t t0 = now_ns();
    if (count == 0) return QRM_OK;
    // Register the caller's whole input and output ranges once, before the shard
    // threads start: per-shard registration of sub-ranges of one pageable buffer
    // would overlap at shared boundary pages (and one shard's unregister would
    // pull the page from under its neighbour).
    const int64_t in_bytes = (count - 1) * stride + static_cast<int64_t>(w) * h * 3;
    bool reg_in = false, reg_out = false;
    auto unreg = on_exit([&] {
        if (reg_in) cudaHostUnregister(const_cast<uint8_t*>(images));
        if (reg_out) cudaHostUnregister(out);
    });
    if ((s = set_device(ctxs[0]->device)) != QRM_OK) return s;
    cudaPointerAttributes attr{};
    if (cudaPointerGetAttributes(&attr, images) != cudaSuccess || attr.type != cudaMemoryTypeHost) {
        cudaGetLastError();
        QRM_CUDA(cudaHostRegister(const_cast<uint8_t*>(images), in_bytes,
                                  cudaHostRegisterMapped | cudaHostRegisterPortable | cudaHostRegisterReadOnly));
        reg_in = true;
    }
    if (cudaPointerGetAttributes(&attr, out) != cudaSuccess || attr.type != cudaMemoryTypeHost) {
        cudaGetLastError();
        QRM_CUDA(cudaHostRegister(out, sizeof(qrm_record) * count, cudaHostRegisterPortable));
        reg_out = true;
    }
    std::vector<qrm_status> st(nctx, QRM_OK);
    std::vector<std::string> err(nctx);
    std::vector<qrm_host_stats> part(nctx);
    auto run = [&](int i) {
        pin_thread_to_device(ctxs[i]->device);  // each shard's host thread on its GPU's NUMA node
        const int64_t b = count * i / nctx, e = count * (i + 1) / nctx;
        st[i] = qrm_detect_host(ctxs[i], images + b * stride, e - b, w, h, stride, first_draw + static_cast<uint64_t>(b),
                                out + b, plan, mode, &part[i]);
        if (st[i] != QRM_OK) err[i] = g_err;  // thread-local: carried to the caller below
    };
    std::vector<std::thread> th;  // one thread per shard (the caller's own affinity stays untouched)
    for (int i = 0; i < nctx; ++i) th.emplace_back(run, i);
    for (auto& t : th) t.join();
    for (int i = 0; i < nctx; ++i)
        if (st[i] != QRM_OK) return fail(st[i], "shard " + std::to_string(i) + ": " + err[i]);
    if (stats) {
        *stats = qrm_host_stats{};
        for (const auto& p : part) {
            stats->h2d_bytes += p.h2d_bytes;
            stats->d2h_bytes += p.d2h_bytes;
            stats->minibatches += p.minibatches;
            stats->kernel_launches += p.kernel_launches;
        }
        stats->wall_ms = static_cast<double>(now_ns() - t0) / 1e6;
    }
    return QRM_OK;
}

QRM_EXPORT qrm_status qrm_preprocess_host(const uint8_t* image, int w, int h, float* out) {
    // Full preprocess (transforms.cpp:42-47) on the device: the 256x256 crop is
    // gathered as one "tile" of size 256 with the fixed strategy.
    if (!image || !out) return fail(QRM_INVALID_INPUT, "null argument");
    if (w <= 0 || h <= 0) return fail(QRM_INVALID_INPUT, "image dimensions must be positive");
    int up, sw, sh, xo, yo;
    geometry(w, h, up, sw, sh, xo, yo);
    const int64_t bytes = static_cast<int64_t>(w) * h * 3;
    const int64_t K = 256 * 256 * 3;
    uint8_t *dimg = nullptr, *dwin = nullptr;
    GatherDesc* dd = nullptr;
    QRM_CUDA(cudaMalloc(&dimg, bytes));
    QRM_CUDA(cudaMalloc(&dwin, K));
    QRM_CUDA(cudaMalloc(&dd, sizeof(GatherDesc)));
    QRM_CUDA(cudaMemcpy(dimg, image, bytes, cudaMemcpyHostToDevice));
    GatherDesc d{dimg, w, h, up, sw, sh, xo, yo, 0, 0};
    QRM_CUDA(cudaMemcpy(dd, &d, sizeof d, cudaMemcpyHostToDevice));
    QRM_LAUNCH(launch_gather_windows(dd, 1, 256, dwin, nullptr));
    std::vector<uint8_t> win(K);
    QRM_CUDA(cudaMemcpy(win.data(), dwin, K, cudaMemcpyDeviceToHost));
    cudaFree(dimg);
    cudaFree(dwin);
    cudaFree(dd);
    for (int64_t i = 0; i < K; ++i) out[i] = static_cast<float>(win[i] / 127.5 - 1.0);  // image.cpp:36
    return QRM_OK;
}

// Device codebooks (row f1), one per (device, code), created on first use:
// 2^22 slots (64 MiB of keys + values, 4 MiB of error counts), keys all-ones.
static std::mutex g_codebook_mu;
static std::map<std::tuple<int, int, int, int>, CodebookTable> g_codebooks;
constexpr uint64_t kCodebookSlots = 1ull << 22;

static qrm_status codebook_for(int dev, int m, int n, int k, cudaStream_t st, CodebookTable* out) {
    std::lock_guard<std::mutex> g(g_codebook_mu);
    auto key = std::make_tuple(dev, m, n, k);
    auto it = g_codebooks.find(key);
    if (it == g_codebooks.end()) {
        CodebookTable c{nullptr, nullptr, nullptr, kCodebookSlots - 1};
        QRM_CUDA(cudaMalloc(&c.keys, sizeof(uint64_t) * kCodebookSlots));
        QRM_CUDA(cudaMalloc(&c.vals, sizeof(uint64_t) * kCodebookSlots));
        QRM_CUDA(cudaMalloc(&c.nerr, kCodebookSlots));
        QRM_CUDA(cudaMemsetAsync(c.keys, 0xFF, sizeof(uint64_t) * kCodebookSlots, st));
        it = g_codebooks.emplace(key, c).first;
    }
    *out = it->second;
    return QRM_OK;
}

QRM_EXPORT qrm_status qrm_rs_decode_packed_device(int m, int n, int k, const uint64_t* words, int64_t count,
                                                  uint64_t* cw_out, int8_t* nerr_out, int algo, void* stream) {
    const std::string e = check_code(m, n, k);
    if (!e.empty()) return fail(QRM_INVALID_INPUT, e);
    if (n * m > 64) return fail(QRM_INVALID_INPUT, "packed words need n*m <= 64");
    if (count < 0) return fail(QRM_INVALID_INPUT, "negative count");
    const int t = (n - k) / 2;
    if (algo == 0) algo = (t == 1 && n - k <= 3) ? 1 : 2;
    if (algo < 1 || algo > 3) return fail(QRM_INVALID_INPUT, "algo must be 0 (auto), 1, 2 or 3");
    if (algo == 1 && !(t == 1 && n - k <= 3)) return fail(QRM_INVALID_INPUT, "thread decoder needs t = 1");
    if (algo == 3 && n * m >= 64) return fail(QRM_INVALID_INPUT, "the device codebook needs n*m < 64");
    if (t > 8) return fail(QRM_INVALID_INPUT, "packed warp decoder supports t <= 8");
    const RsTables* tab;
    qrm_status s = rs_tables_for(m, n, k, &tab);
    if (s != QRM_OK) return s;
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    CodebookTable cache{nullptr, nullptr, nullptr, 0};
    if (algo == 3) {
        s = codebook_for(dev, m, n, k, as_stream(stream), &cache);
        if (s != QRM_OK) return s;
    }
    QRM_LAUNCH(launch_rs_packed(tab, m, n, n - k, t, algo == 3 ? 2 : algo, words, count, cw_out, nerr_out, sms,
                                as_stream(stream), cache));
    return QRM_OK;
}

QRM_EXPORT qrm_status qrm_rs_codebook_clear(int m, int n, int k, void* stream) {
    const std::string e = check_code(m, n, k);
    if (!e.empty()) return fail(QRM_INVALID_INPUT, e);
    int dev = 0;
    cudaGetDevice(&dev);
    CodebookTable cache{nullptr, nullptr, nullptr, 0};
    qrm_status s = codebook_for(dev, m, n, k, as_stream(stream), &cache);
    if (s != QRM_OK) return s;
    QRM_CUDA(cudaMemsetAsync(cache.keys, 0xFF, sizeof(uint64_t) * (cache.mask + 1), as_stream(stream)));
    return QRM_OK;
}

QRM_EXPORT qrm_status qrm_rs_decode_symbols_device(int m, int n, int k, const uint8_t* recv, int64_t count,
                                                   uint8_t* cw_out, int8_t* nerr_out, void* stream) {
    const std::string e = check_code(m, n, k);
    if (!e.empty()) return fail(QRM_INVALID_INPUT, e);
    if (count < 0) return fail(QRM_INVALID_INPUT, "negative count");
    const int t = (n - k) / 2;
    if (t > 31) return fail(QRM_INVALID_INPUT, "symbol decoder supports t <= 31");
    const RsTables* tab;
    qrm_status s = rs_tables_for(m, n, k, &tab);
    if (s != QRM_OK) return s;
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    QRM_LAUNCH(launch_rs_symbols(tab, n, t, recv, count, cw_out, nerr_out, sms, as_stream(stream)));
    return QRM_OK;
}

// RS stress words for the RS-only benchmark (device): message, received word,
// injected error count.
QRM_EXPORT qrm_status qrm_rs_stress_device(int m, int n, int k, uint64_t seed, int64_t count, uint64_t* msg,
                                           uint64_t* words, int8_t* nerr_true, void* stream) {
    const std::string e = check_code(m, n, k);
    if (!e.empty()) return fail(QRM_INVALID_INPUT, e);
    if (n * m > 64 || n > 32) return fail(QRM_INVALID_INPUT, "stress words need n*m <= 64");
    const RsTables* tab;
    qrm_status s = rs_tables_for(m, n, k, &tab);
    if (s != QRM_OK) return s;
    auto masks = build_encoder_masks(m, n, k);
    uint64_t* dm = nullptr;
    QRM_CUDA(cudaMalloc(&dm, sizeof(uint64_t) * std::max<size_t>(1, masks.size())));
    QRM_CUDA(cudaMemcpy(dm, masks.data(), sizeof(uint64_t) * masks.size(), cudaMemcpyHostToDevice));
    QRM_LAUNCH(launch_rs_stress(tab, dm, seed, count, msg, words, nerr_true, as_stream(stream)));
    QRM_CUDA(cudaStreamSynchronize(as_stream(stream)));
    cudaFree(dm);
    return QRM_OK;
}

QRM_EXPORT qrm_status qrm_rs_stress_symbols_device(int m, int n, int k, uint64_t seed, int64_t count,
                                                   uint8_t* true_cw, uint8_t* recv, int8_t* nerr_true, void* stream) {
    const std::string e = check_code(m, n, k);
    if (!e.empty()) return fail(QRM_INVALID_INPUT, e);
    if (m > 8) return fail(QRM_INVALID_INPUT, "symbol stress words need m <= 8");
    const int r = n - k;
    if (static_cast<int64_t>(k) * r > 96 * 1024) return fail(QRM_INVALID_INPUT, "parity generator exceeds 96 KiB");
    if (count < 0) return fail(QRM_INVALID_INPUT, "negative count");
    const RsTables* tab;
    qrm_status s = rs_tables_for(m, n, k, &tab);
    if (s != QRM_OK) return s;
    // parity generator: G[j][c] = parity symbol c of rs_encode(unit message j) (encoding is GF-linear)
    std::vector<uint8_t> gpar(static_cast<size_t>(k) * r);
    std::vector<uint16_t> msg(k, 0);
    for (int j = 0; j < k; ++j) {
        msg[j] = 1;
        const auto cw = encode_symbols(m, n, k, msg);
        msg[j] = 0;
        for (int c = 0; c < r; ++c) gpar[static_cast<size_t>(j) * r + c] = static_cast<uint8_t>(cw[k + c]);
    }
    uint8_t* dg = nullptr;
    QRM_CUDA(cudaMalloc(&dg, std::max<size_t>(1, gpar.size())));
    QRM_CUDA(cudaMemcpy(dg, gpar.data(), gpar.size(), cudaMemcpyHostToDevice));
    QRM_LAUNCH(launch_rs_stress_symbols(tab, dg, k, r, seed, count, true_cw, recv, nerr_true, as_stream(stream)));
    QRM_CUDA(cudaStreamSynchronize(as_stream(stream)));
    cudaFree(dg);
    return QRM_OK;
}

QRM_EXPORT qrm_status qrm_patterns_device(uint64_t key_seed, int n_bits, int l, int8_t* out, void* stream) {
    if (n_bits <= 0 || n_bits > kMaxNBits || l <= 0) return fail(QRM_INVALID_INPUT, "bad pattern geometry");
    const int K = 3 * l * l;
    int32_t* cs = nullptr;
    QRM_CUDA(cudaMalloc(&cs, sizeof(int32_t) * kMaxNBits));
    int8_t* tmp = nullptr;
    QRM_CUDA(cudaMalloc(&tmp, static_cast<size_t>(kMaxNBits) * K));
    QRM_LAUNCH(launch_build_patterns(key_seed, n_bits, K, K, tmp, cs, as_stream(stream)));
    QRM_CUDA(cudaMemcpyAsync(out, tmp, static_cast<size_t>(n_bits) * K, cudaMemcpyDeviceToDevice, as_stream(stream)));
    QRM_CUDA(cudaStreamSynchronize(as_stream(stream)));
    cudaFree(cs);
    cudaFree(tmp);
    return QRM_OK;
}

QRM_EXPORT qrm_status qrm_make_corpus_device(const qrm_config* cfg, uint64_t first_seed, int64_t count, int w, int h,
                                             int embed, uint8_t* out, void* stream) {
    if (!cfg) return fail(QRM_INVALID_INPUT, "null config");
    if (w <= 0 || h <= 0 || count < 0) return fail(QRM_INVALID_INPUT, "bad corpus geometry");
    float* delta = nullptr;
    const int l = cfg->tile_size;
    if (embed) {
        const std::string ce = check_code(cfg->symbol_bits, cfg->n, cfg->k);
        if (!ce.empty()) return fail(QRM_INVALID_INPUT, ce);
        const int nbits = cfg->n * cfg->symbol_bits, kbits = cfg->k * cfg->symbol_bits;
        if (nbits > 64) return fail(QRM_INVALID_INPUT, "corpus embedding supports codewords up to 64 bits");
        if (!cfg->key_message) return fail(QRM_INVALID_INPUT, "key message missing");
        uint64_t msg = 0;
        for (int i = 0; i < kbits; ++i) msg = (msg << 1) | (cfg->key_message[i] & 1);
        const uint64_t cw = encode_packed(cfg->symbol_bits, cfg->n, cfg->k, msg);
        QRM_CUDA(cudaMalloc(&delta, sizeof(float) * 3 * l * l));
        QRM_LAUNCH(launch_residual(cfg->key_seed, nbits, 3 * l * l, cw, delta, as_stream(stream)));
    }
    QRM_LAUNCH(launch_corpus(first_seed, count, w, h, l, embed, static_cast<float>(cfg->alpha), delta, out,
                             as_stream(stream)));
    if (delta) {
        QRM_CUDA(cudaStreamSynchronize(as_stream(stream)));
        cudaFree(delta);
    }
    return QRM_OK;
}

}  // extern "C"

namespace {

// cuTensorMapEncodeTiled through the runtime's driver entry point (no -lcuda).
qrm_status tensor_map_encoder(PFN_cuTensorMapEncodeTiled_v12000* out) {
    // resolved once per process (thread-safe static initialisation)
    static const PFN_cuTensorMapEncodeTiled_v12000 encode = [] {
        cudaDriverEntryPointQueryResult q;
        void* fn = nullptr;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) != cudaSuccess ||
            q != cudaDriverEntryPointSuccess) {
            cudaGetLastError();
            fn = nullptr;
        }
        return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
    }();
    if (!encode) return fail(QRM_CUDA_ERROR, "cuTensorMapEncodeTiled unavailable");
    *out = encode;
    return QRM_OK;
}

qrm_status encode_act_tmap(CUtensorMap* map, CUtensorMap* store_map, void* base, int64_t tiles) {
    PFN_cuTensorMapEncodeTiled_v12000 encode = nullptr;
    if (qrm_status s = tensor_map_encoder(&encode); s != QRM_OK) return s;
    // activations NHWC bf16 [T][64 y][64 x][64 c]; box = 4 rows of 64 pixels
    const cuuint64_t dims[4] = {64, 64, 64, static_cast<cuuint64_t>(tiles)};
    const cuuint64_t strides[3] = {64 * 2, 64 * 64 * 2, 64 * 64 * 64 * 2};
    const cuuint32_t box[4] = {64, 64, 4, 1};
    const cuuint32_t estr[4] = {1, 1, 1, 1};
    const CUresult r = encode(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, base, dims, strides, box, estr,
                              CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                              CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) return fail(QRM_CUDA_ERROR, "cuTensorMapEncodeTiled failed (" + std::to_string(r) + ")");
    // store view of the same buffer: [T*4096 pixels][64 c]; box = 32 pixels (one
    // epilogue warp's slab), written from a 128B-swizzled staging slab
    const cuuint64_t sdims[2] = {64, static_cast<cuuint64_t>(tiles) * 4096};
    const cuuint64_t sstrides[1] = {64 * 2};
    const cuuint32_t sbox[2] = {64, 32};
    const CUresult r2 = encode(store_map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, base, sdims, sstrides, sbox, estr,
                               CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                               CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r2 != CUDA_SUCCESS) return fail(QRM_CUDA_ERROR, "cuTensorMapEncodeTiled (store) failed (" + std::to_string(r2) + ")");
    return QRM_OK;
}

// One 64->64 conv layer: the CTA-pair kernel (cta_group::2, M = 256; 237 us per
// 1024 tiles against 285 us for the single-CTA kernel) unless the context was
// created with QRM_CONV_PAIR=0.
cudaError_t conv64_layer(const qrm_ctx* c, const CUtensorMap& tmap, const CUtensorMap& tmap_out,
                         const HiddenLayerParams& p, cudaStream_t st) {
    return c->conv_pair ? launch_conv64_pair(tmap, tmap_out, p, c->sms, st)
                        : launch_conv64(tmap, tmap_out, p, c->sms, st);
}

qrm_status hidden_prepare(qrm_ctx* c, uint64_t seed, int64_t tiles, cudaStream_t st) {
    auto& H = c->hid;
    if (!H.w_sw) {
        QRM_CUDA(cudaMalloc(&H.w_sw, sizeof(__nv_bfloat16) * 8 * 9 * 64 * 64));
        QRM_CUDA(cudaMalloc(&H.bias, sizeof(float) * 9 * 64));
        QRM_CUDA(cudaMalloc(&H.w0, sizeof(float) * 64 * 32));
        QRM_CUDA(cudaMalloc(&H.wl, sizeof(float) * 64 * 64));
        QRM_CUDA(cudaMalloc(&H.bl, sizeof(float) * 64));
    }
    if (!H.ready || H.seed != seed) {
        QRM_LAUNCH(launch_hidden_prep(seed, c->nbits, H.w_sw, H.bias, H.w0, H.wl, H.bl, st));
        H.ready = true;
        H.seed = seed;
    }
    if (tiles > H.tiles_cap) {
        for (auto& a : H.act) cudaFree(a);
        cudaFree(H.pool);
        const size_t act_bytes = sizeof(__nv_bfloat16) * 64 * 64 * 64 * static_cast<size_t>(tiles);
        QRM_CUDA(cudaMalloc(&H.act[0], act_bytes));
        QRM_CUDA(cudaMalloc(&H.act[1], act_bytes));
        QRM_CUDA(cudaMalloc(&H.pool, sizeof(float) * kHiddenBlocksPerTile * 64 * tiles));
        qrm_status s;
        for (int i = 0; i < 2; ++i)
            if ((s = encode_act_tmap(&H.tmap[i], &H.tmap_st[i], H.act[i], tiles)) != QRM_OK) return s;
        H.tiles_cap = tiles;
    }
    return QRM_OK;
}

// The windows of images [off, off + n) of a batch source.
WindowSource slice_source(const WindowSource& src, int64_t off, int K) {
    WindowSource s = src;
    if (src.direct) {
        s.base = src.base + off * src.image_stride;
        s.first_draw = src.first_draw + static_cast<uint64_t>(off);
    } else {
        s.base = src.base + off * static_cast<int64_t>(K);
    }
    return s;
}

// Learned extractor over `count` windows: conv0 -> 8 x conv64 -> head (pool,
// linear, harden, t = 1 RS + verify) -> finish (general-t codes), in chunks of
// at most kConvChunk tiles (activation ping-pong buffers: 2 x 512 KB per tile).
qrm_status hidden_run(qrm_ctx* c, Workspace& W, const WindowSource& src, int64_t count, qrm_record* out,
                      float* logits, cudaStream_t st) {
    constexpr int64_t kConvChunk = 8192;
    if (c->l != 64) return fail(QRM_INVALID_INPUT, "the conv extractor is defined on 64x64 tiles");
    qrm_status s;
    if ((s = hidden_prepare(c, c->conv_seed, std::min(count, kConvChunk), st)) != QRM_OK) return s;
    auto& H = c->hid;
    for (int64_t off = 0; off < count; off += kConvChunk) {
        const int64_t n = std::min(kConvChunk, count - off);
        const WindowSource cs = slice_source(src, off, c->K);
        const bool pair = c->conv_pair;
        // the pair kernel's last layer folds the linear layer into its epilogue
        // (QRM_CONV_FUSE_LINEAR=0: channel partials + hidden_head_kernel instead)
        const bool fuse_linear = pair && c->conv_fuse_linear;
        Conv0Params p0{cs, n, c->K, H.w0, H.bias, H.act[0]};
        QRM_LAUNCH(launch_conv0(p0, H.tmap_st[0], c->sms, st));
        for (int j = 1; j < kHiddenLayers; ++j) {
            HiddenLayerParams lp{};
            lp.w_swizzled = H.w_sw + static_cast<int64_t>(j - 1) * 9 * 64 * 64;
            lp.bias = H.bias + j * 64;
            lp.last = j == kHiddenLayers - 1;
            lp.act_out = lp.last ? nullptr : H.act[j & 1];
            lp.pool_out = lp.last ? H.pool : nullptr;
            lp.tiles = n;
            if (lp.last && fuse_linear) {
                lp.fuse_linear = 1;
                lp.wl = H.wl;
                lp.nbits = c->nbits;
            }
            QRM_LAUNCH(conv64_layer(c, H.tmap[(j - 1) & 1], H.tmap_st[j & 1], lp, st));
        }
        HeadParams hp{};
        hp.pool = H.pool;
        hp.wl = H.wl;
        hp.bl = H.bl;
        hp.tiles = n;
        hp.nbits = c->nbits;
        hp.kbits = c->kbits;
        hp.tau_msg = c->tau_msg;
        hp.tau_raw = c->tau_raw;
        hp.fuse_t1 = (c->t == 1 && c->n - c->k <= 3) ? 1 : 0;
        hp.key_cw = c->key_cw;
        hp.key_msg = c->key_msg;
        hp.rs = c->d_rs;
        hp.logits = logits ? logits + off * c->nbits : nullptr;
        hp.out = out + off;
        hp.pending_count = W.pending_count;
        hp.pending = W.pending;
        if (fuse_linear) QRM_LAUNCH(launch_hidden_sign(hp, st));
        else QRM_LAUNCH(launch_hidden_head(hp, st));
        DetectParams fp = base_params(c, W, n, out + off, nullptr, nullptr);
        fp.src = cs;
        if (!fp.fuse_t1) QRM_LAUNCH(launch_detect_finish(fp, std::max(1, c->t), c->sms, st));  // general-t codes
    }
    return QRM_OK;
}

}  // namespace

extern "C" {

QRM_EXPORT qrm_status qrm_hidden_detect_device(qrm_ctx* c, const uint8_t* images, int64_t count, int w, int h,
                                               int64_t stride, uint64_t first_draw, uint64_t weight_seed,
                                               float* logits, qrm_record* out, void* stream) {
    qrm_status s = check_uniform(c, images, count, w, h, stride);
    if (s != QRM_OK) return s;
    if (count > 0 && !out) return fail(QRM_INVALID_INPUT, "null record buffer");
    if (c->l != 64) return fail(QRM_INVALID_INPUT, "the conv extractor is defined on 64x64 tiles");
    if ((s = set_device(c->device)) != QRM_OK) return s;
    if (count == 0) return QRM_OK;
    cudaStream_t st = as_stream(stream);
    Workspace& W = c->ws[0];
    const uint64_t keep = c->conv_seed;
    c->conv_seed = weight_seed;
    if ((s = workspace_reserve(W, count)) != QRM_OK) return s;
    WindowSource src;
    if ((s = window_source(c, W, images, count, w, h, stride, first_draw, st, src)) == QRM_OK)
        s = hidden_run(c, W, src, count, out, logits, st);
    c->conv_seed = keep;
    return s;
}

QRM_EXPORT qrm_status qrm_extract_tiles_device(qrm_ctx* c, const uint8_t* images, int64_t count, int w, int h,
                                               int64_t stride, uint64_t first_draw, int channels, void* out,
                                               void* stream) {
    // preprocess -> select_tile -> extract_tile -> normalize as bf16 NHWC tiles.
    qrm_status s = check_uniform(c, images, count, w, h, stride);
    if (s != QRM_OK) return s;
    if (c->l != 64) return fail(QRM_INVALID_INPUT, "bf16 tile extraction is built for 64x64 tiles");
    if (channels != 3 && channels != 4) return fail(QRM_INVALID_INPUT, "channels must be 3 or 4");
    if (count > 0 && !out) return fail(QRM_INVALID_INPUT, "null output buffer");
    if (count >= (int64_t{1} << 31)) return fail(QRM_INVALID_INPUT, "too many tiles for one launch");
    if ((s = set_device(c->device)) != QRM_OK) return s;
    if (count == 0) return QRM_OK;
    cudaStream_t st = as_stream(stream);
    Workspace& W = c->ws[0];
    WindowSource src;
    if ((s = window_source(c, W, images, count, w, h, stride, first_draw, st, src)) != QRM_OK) return s;
    PFN_cuTensorMapEncodeTiled_v12000 encode = nullptr;
    if ((s = tensor_map_encoder(&encode)) != QRM_OK) return s;
    // u8 images viewed as [count][rows][row bytes]; box = one 64 x 192-B window
    const bool direct = src.direct != 0;
    const cuuint64_t dims[3] = {static_cast<cuuint64_t>(direct ? w * 3 : 192), static_cast<cuuint64_t>(direct ? h : 64),
                                static_cast<cuuint64_t>(count)};
    const cuuint64_t strides[2] = {static_cast<cuuint64_t>(direct ? w * 3 : 192),
                                   static_cast<cuuint64_t>(direct ? stride : c->K)};
    const cuuint32_t box[3] = {192, 64, 1};
    const cuuint32_t estr[3] = {1, 1, 1};
    CUtensorMap map;
    const CUresult r = encode(&map, CU_TENSOR_MAP_DATA_TYPE_UINT8, 3, const_cast<uint8_t*>(src.base), dims, strides,
                              box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                              // 64-B fills: a 192-B row at a 64-B offset, no over-read
                              CU_TENSOR_MAP_L2_PROMOTION_L2_64B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) return fail(QRM_CUDA_ERROR, "cuTensorMapEncodeTiled (tiles) failed (" + std::to_string(r) + ")");
    TileBf16Params p{src, count, c->K, channels, static_cast<uint16_t*>(out)};
    QRM_LAUNCH(launch_tile_bf16(map, p, c->sms, st));
    return QRM_OK;
}

QRM_EXPORT qrm_status qrm_ctx_set_transfer_split(qrm_ctx* c, double zero_copy_fraction) {
    if (!c) return fail(QRM_INVALID_INPUT, "null context");
    if (!(zero_copy_fraction >= 0.0 && zero_copy_fraction <= 1.0))
        return fail(QRM_INVALID_INPUT, "zero-copy fraction must be in [0, 1]");
    c->hybrid_fraction = zero_copy_fraction;
    return QRM_OK;
}

QRM_EXPORT qrm_status qrm_ctx_set_extractor(qrm_ctx* c, int kind, uint64_t weight_seed) {
    if (!c) return fail(QRM_INVALID_INPUT, "null context");
    if (kind != QRM_EXTRACTOR_SPREAD_SPECTRUM && kind != QRM_EXTRACTOR_CONV)
        return fail(QRM_INVALID_INPUT, "unknown extractor kind");
    if (kind == QRM_EXTRACTOR_CONV && c->l != 64)
        return fail(QRM_INVALID_INPUT, "the conv extractor is defined on 64x64 tiles");
    c->extractor = kind;
    c->conv_seed = weight_seed;
    return QRM_OK;
}

QRM_EXPORT qrm_status qrm_hidden_debug_activation(qrm_ctx* c, const uint8_t* images, int64_t count, int w, int h,
                                                  int64_t stride, uint64_t first_draw, uint64_t weight_seed,
                                                  int stop_after, void* out, void* stream) {
    qrm_status s = check_uniform(c, images, count, w, h, stride);
    if (s != QRM_OK) return s;
    if (c->l != 64 || stop_after < 0 || stop_after > kHiddenLayers - 1 || !out)
        return fail(QRM_INVALID_INPUT, "bad debug request");
    if ((s = set_device(c->device)) != QRM_OK) return s;
    cudaStream_t st = as_stream(stream);
    Workspace& W = c->ws[0];
    if ((s = hidden_prepare(c, weight_seed, count, st)) != QRM_OK) return s;
    WindowSource src;
    if ((s = window_source(c, W, images, count, w, h, stride, first_draw, st, src)) != QRM_OK) return s;
    auto& H = c->hid;
    Conv0Params p0{src, count, c->K, H.w0, H.bias, H.act[0]};
    QRM_LAUNCH(launch_conv0(p0, H.tmap_st[0], c->sms, st));
    for (int j = 1; j <= stop_after; ++j) {
        HiddenLayerParams lp{};
        lp.w_swizzled = H.w_sw + static_cast<int64_t>(j - 1) * 9 * 64 * 64;
        lp.bias = H.bias + j * 64;
        lp.last = j == kHiddenLayers - 1;
        lp.act_out = lp.last ? nullptr : H.act[j & 1];
        lp.pool_out = lp.last ? H.pool : nullptr;
        lp.tiles = count;
        QRM_LAUNCH(conv64_layer(c, H.tmap[(j - 1) & 1], H.tmap_st[j & 1], lp, st));
    }
    if (stop_after == kHiddenLayers - 1)
        QRM_CUDA(cudaMemcpyAsync(out, H.pool, sizeof(float) * kHiddenBlocksPerTile * 64 * count,
                                 cudaMemcpyDeviceToDevice, st));
    else
        QRM_CUDA(cudaMemcpyAsync(out, H.act[stop_after & 1], sizeof(__nv_bfloat16) * 64 * 64 * 64 * count,
                                 cudaMemcpyDeviceToDevice, st));
    return QRM_OK;
}

QRM_EXPORT qrm_status qrm_extract_float_host(uint64_t key_seed, int n_bits, int l, const float* tile, double* soft) {
    if (!tile || !soft || n_bits <= 0 || l <= 0) return fail(QRM_INVALID_INPUT, "bad extract arguments");
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) return fail(QRM_NO_DEVICE, "no CUDA device available");
    const int K = 3 * l * l;
    float* dt = nullptr;
    double* ds = nullptr;
    QRM_CUDA(cudaMalloc(&dt, sizeof(float) * K));
    QRM_CUDA(cudaMalloc(&ds, sizeof(double) * n_bits));
    QRM_CUDA(cudaMemcpy(dt, tile, sizeof(float) * K, cudaMemcpyHostToDevice));
    QRM_LAUNCH(launch_extract_float(key_seed, n_bits, K, dt, ds, nullptr));
    QRM_CUDA(cudaMemcpy(soft, ds, sizeof(double) * n_bits, cudaMemcpyDeviceToHost));
    cudaFree(dt);
    cudaFree(ds);
    return QRM_OK;
}

QRM_EXPORT qrm_status qrm_resample_host(const uint8_t* image, int w, int h, int upscale, int sw, int sh, int x_off,
                                        int y_off, int out_w, int out_h, int normalize, void* out) {
    if (!image || !out || w <= 0 || h <= 0 || out_w <= 0 || out_h <= 0)
        return fail(QRM_INVALID_INPUT, "bad resample arguments");
    if (!upscale && (x_off < 0 || y_off < 0 || x_off + out_w > w || y_off + out_h > h))
        return fail(QRM_INVALID_INPUT, "window outside the image");
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) return fail(QRM_NO_DEVICE, "no CUDA device available");
    const int64_t bytes = static_cast<int64_t>(w) * h * 3;
    const int64_t n = static_cast<int64_t>(out_w) * out_h * 3;
    const int64_t ob = n * (normalize ? sizeof(float) : 1);
    uint8_t* dimg = nullptr;
    void* dout = nullptr;
    QRM_CUDA(cudaMalloc(&dimg, bytes));
    QRM_CUDA(cudaMalloc(&dout, ob));
    QRM_CUDA(cudaMemcpy(dimg, image, bytes, cudaMemcpyHostToDevice));
    GatherDesc d{dimg, w, h, upscale, sw, sh, x_off, y_off, 0, 0};
    QRM_LAUNCH(launch_resample(d, out_w, out_h, normalize, dout, nullptr));
    QRM_CUDA(cudaMemcpy(out, dout, ob, cudaMemcpyDeviceToHost));
    cudaFree(dimg);
    cudaFree(dout);
    return QRM_OK;
}

QRM_EXPORT qrm_status qrm_attack_device(const uint8_t* images, int64_t count, int w, int h, int64_t stride, int op,
                                        double param, void* out, int64_t out_stride, int* out_w, int* out_h,
                                        void* stream) {
    // Argument checks, output geometry and host-side constants follow
    // apply_attack (transforms.cpp:289-362) and its helpers.
    if (count < 0 || w <= 0 || h <= 0 || !out_w || !out_h) return fail(QRM_INVALID_INPUT, "bad attack arguments");
    AttackParams p{};
    p.in = images;
    p.in_stride = stride;
    p.w = w;
    p.h = h;
    p.count = count;
    p.op = op;
    p.param = param;
    p.sw = w;
    p.sh = h;
    int ow = w, oh = h;
    int stages = 1;  // resize: two resample passes
    int dw = 0, dh = 0;
    auto crop_to = [&](int cw, int ch) -> qrm_status {
        if (cw > w || ch > h) return fail(QRM_INVALID_INPUT, "crop window larger than image");
        ow = cw;
        oh = ch;
        p.x_off = (w - cw) / 2;
        p.y_off = (h - ch) / 2;
        return QRM_OK;
    };
    qrm_status s = QRM_OK;
    switch (op) {
        case QRM_ATTACK_CENTERCROP: {
            const int side = static_cast<int>(param);
            if (side <= 0) return fail(QRM_INVALID_INPUT, "centercrop size must be positive");
            s = crop_to(std::min(side, w), std::min(side, h));
            break;
        }
        case QRM_ATTACK_RESIZETO: {
            const int side = static_cast<int>(param);
            if (side <= 0) return fail(QRM_INVALID_INPUT, "resizeto size must be positive");
            ow = oh = side;
            p.resize = 1;
            p.sw = p.sh = side;
            break;
        }
        case QRM_ATTACK_NORMALIZE: p.normalize = 1; break;
        case QRM_ATTACK_CROP: {
            if (param <= 0.0 || param > 1.0) return fail(QRM_INVALID_INPUT, "crop fraction must be in (0, 1]");
            const double f = std::sqrt(param);
            s = crop_to(std::max(1, static_cast<int>(std::lround(w * f))), std::max(1, static_cast<int>(std::lround(h * f))));
            break;
        }
        case QRM_ATTACK_RESIZE:
            if (param <= 0.0 || param >= 1.0) {
                if (param != 1.0) return fail(QRM_INVALID_INPUT, "resize factor must be in (0, 1)");
                break;  // identity
            }
            dw = std::max(1, static_cast<int>(std::lround(w * param)));
            dh = std::max(1, static_cast<int>(std::lround(h * param)));
            stages = 2;
            break;
        case QRM_ATTACK_BRIGHTNESS:
            if (param < 0.0) return fail(QRM_INVALID_INPUT, "brightness factor must be nonnegative");
            break;
        case QRM_ATTACK_CONTRAST:
            if (param < 0.0) return fail(QRM_INVALID_INPUT, "contrast factor must be nonnegative");
            break;
        case QRM_ATTACK_SATURATION:
            if (param < 0.0) return fail(QRM_INVALID_INPUT, "saturation factor must be nonnegative");
            break;
        case QRM_ATTACK_SHARPNESS:
            if (param < 0.0) return fail(QRM_INVALID_INPUT, "sharpness factor must be nonnegative");
            break;
        case QRM_ATTACK_BLUR:
        case QRM_ATTACK_OVERLAY_TEXT: break;
        case QRM_ATTACK_JPEG_APPROX:
            if (param <= 0.0 || param > 100.0) return fail(QRM_INVALID_INPUT, "jpeg_approx quality must be in (0, 100]");
            break;
        default: return fail(QRM_INVALID_INPUT, "unknown transform op");
    }
    if (s != QRM_OK) return s;
    *out_w = ow;
    *out_h = oh;
    if (!out || count == 0) return QRM_OK;
    if (!images) return fail(QRM_INVALID_INPUT, "null image pointer");
    if (stride < static_cast<int64_t>(w) * h * 3) return fail(QRM_INVALID_INPUT, "image stride smaller than an image");
    const int64_t out_bytes = static_cast<int64_t>(ow) * oh * 3 * (op == QRM_ATTACK_NORMALIZE ? 4 : 1);
    if (out_stride < out_bytes) return fail(QRM_INVALID_INPUT, "output stride smaller than an output image");
    cudaStream_t st = as_stream(stream);
    p.out = static_cast<uint8_t*>(out);
    p.out_stride = out_stride;
    p.ow = ow;
    p.oh = oh;
    // host libm constants, exactly as the reference evaluates them
    p.kC = 1.0;
    p.kE = std::exp(-0.5);
    p.kD = std::exp(-1.0);
    p.kSum = p.kC + 4.0 * p.kE + 4.0 * p.kD;
    double* dtmp = nullptr;  // pivots / jpeg tables
    uint8_t* mid = nullptr;  // resize: the downscaled intermediate
    struct Free {
        double*& a;
        uint8_t*& b;
        ~Free() {
            cudaFree(a);
            cudaFree(b);
        }
    } release{dtmp, mid};
    switch (op) {
        case QRM_ATTACK_CENTERCROP: case QRM_ATTACK_RESIZETO: case QRM_ATTACK_NORMALIZE: case QRM_ATTACK_CROP:
            QRM_LAUNCH(launch_attack_resample(p, st));
            break;
        case QRM_ATTACK_RESIZE:
            if (stages == 1) {
                QRM_LAUNCH(launch_attack_resample(p, st));  // factor 1: a copy
            } else {
                // resize_bilinear(resize_bilinear(img, dw, dh), w, h)
                QRM_CUDA(cudaMalloc(&mid, static_cast<size_t>(dw) * dh * 3 * count));
                AttackParams a = p;
                a.out = mid;
                a.out_stride = static_cast<int64_t>(dw) * dh * 3;
                a.ow = a.sw = dw;
                a.oh = a.sh = dh;
                a.resize = 1;
                QRM_LAUNCH(launch_attack_resample(a, st));
                AttackParams b = p;
                b.in = mid;
                b.in_stride = a.out_stride;
                b.w = dw;
                b.h = dh;
                b.resize = 1;
                b.sw = w;
                b.sh = h;
                QRM_LAUNCH(launch_attack_resample(b, st));
            }
            break;
        case QRM_ATTACK_JPEG_APPROX: {
            static const int kQ[64] = {16, 11, 10, 16, 24,  40,  51,  61,  12, 12, 14, 19, 26,  58,  60,  55,
                                       14, 13, 16, 24, 40,  57,  69,  56,  14, 17, 22, 29, 51,  87,  80,  62,
                                       18, 22, 37, 56, 68,  109, 103, 77,  24, 35, 55, 64, 81,  104, 113, 92,
                                       49, 64, 78, 87, 103, 121, 120, 101, 72, 92, 95, 98, 112, 100, 103, 99};
            const double scale = param < 50.0 ? 5000.0 / param : 200.0 - 2.0 * param;
            std::vector<double> tab(128);
            for (int i = 0; i < 64; ++i) tab[64 + i] = std::clamp(std::floor((kQ[i] * scale + 50.0) / 100.0), 1.0, 255.0);
            constexpr double kPi = 3.14159265358979323846;
            for (int u = 0; u < 8; ++u)
                for (int i = 0; i < 8; ++i) tab[u * 8 + i] = std::cos((2 * i + 1) * u * kPi / 16.0);
            QRM_CUDA(cudaMalloc(&dtmp, sizeof(double) * 128));
            QRM_CUDA(cudaMemcpyAsync(dtmp, tab.data(), sizeof(double) * 128, cudaMemcpyHostToDevice, st));
            p.jpeg_cos = dtmp;
            p.jpeg_quant = dtmp + 64;
            p.dct_c0 = std::sqrt(0.125);
            QRM_LAUNCH(launch_attack_jpeg(p, st));
            QRM_CUDA(cudaStreamSynchronize(st));  // the pageable table copy and dtmp outlive no call
            break;
        }
        default:
            if (op == QRM_ATTACK_CONTRAST) {
                QRM_CUDA(cudaMalloc(&dtmp, sizeof(double) * count));
                p.pivot = dtmp;
            }
            QRM_LAUNCH(launch_attack_pixels(p, st));
    }
    if (dtmp || mid) QRM_CUDA(cudaStreamSynchronize(st));  // temporaries are freed on return
    return QRM_OK;
}

QRM_EXPORT qrm_status qrm_allocate_streams(int stages, const double* time, const double* memory, double b0,
                                           int global_batch, int budget, double m_cap, double eps, int stall_cap,
                                           int* streams_out, int* mb_out, double* bottleneck) {
    if (stages <= 0 || !time || !memory || !streams_out || !mb_out || !bottleneck)
        return fail(QRM_INVALID_INPUT, "bad arguments");
    sched::Profile p;
    p.b0 = b0;
    p.time.assign(time, time + stages);
    p.memory.assign(memory, memory + stages);
    sched::Plan plan;
    std::string err;
    const int rc = sched::allocate_streams(p, global_batch, budget, m_cap, eps, stall_cap, plan, err);
    if (rc) return fail(static_cast<qrm_status>(rc), err);
    for (int k = 0; k < stages; ++k) {
        streams_out[k] = plan.streams[k];
        mb_out[k] = plan.minibatch[k];
    }
    *bottleneck = plan.bottleneck;
    return QRM_OK;
}

QRM_EXPORT qrm_status qrm_device_cpus(int device, int* cpus, int capacity, int* count) {
    if (!count || (capacity > 0 && !cpus)) return fail(QRM_INVALID_INPUT, "bad arguments");
    const std::vector<int> v = device_cpus(device);
    *count = static_cast<int>(v.size());
    for (int i = 0; i < capacity && i < static_cast<int>(v.size()); ++i) cpus[i] = v[i];
    return QRM_OK;
}

QRM_EXPORT qrm_status qrm_allocate_streams_sat(int stages, const double* time, const double* memory,
                                               const double* sat, double b0, int global_batch, int budget,
                                               double m_cap, double eps, int stall_cap, int* streams_out,
                                               int* mb_out, double* bottleneck) {
    if (stages <= 0 || !time || !memory || !sat || !streams_out || !mb_out || !bottleneck)
        return fail(QRM_INVALID_INPUT, "bad arguments");
    sched::Profile p;
    p.b0 = b0;
    p.time.assign(time, time + stages);
    p.memory.assign(memory, memory + stages);
    p.sat.assign(sat, sat + stages);
    sched::Plan plan;
    std::string err;
    const int rc = sched::allocate_streams(p, global_batch, budget, m_cap, eps, stall_cap, plan, err);
    if (rc) return fail(static_cast<qrm_status>(rc), err);
    for (int k = 0; k < stages; ++k) {
        streams_out[k] = plan.streams[k];
        mb_out[k] = plan.minibatch[k];
    }
    *bottleneck = plan.bottleneck;
    return QRM_OK;
}

QRM_EXPORT qrm_status qrm_lpt_schedule(int ntasks, const int* ids, const double* lat, const double* mem,
                                       const int* units, int S, double lambda, double m_cap, int b_min, int B,
                                       int capacity, int* p_stream, int* p_id, int* p_units, double* p_lat,
                                       double* p_mem, int* p_mb, int* n_pieces, double* loads, int* m_unit) {
    std::vector<sched::Task> tasks(ntasks);
    for (int i = 0; i < ntasks; ++i) {
        tasks[i].id = ids[i];
        tasks[i].latency = lat[i];
        tasks[i].memory = mem[i];
        tasks[i].units = units[i];
    }
    sched::Schedule out;
    std::string err;
    const int rc = sched::lpt_schedule(tasks, S, lambda, m_cap, b_min, B, out, err);
    if (rc) return fail(static_cast<qrm_status>(rc), err);
    int c = 0;
    for (int st = 0; st < S; ++st) {
        loads[st] = out.loads[st];
        for (const auto& t : out.streams[st]) {
            if (c < capacity) {
                p_stream[c] = st;
                p_id[c] = t.id;
                p_units[c] = t.units;
                p_lat[c] = t.latency;
                p_mem[c] = t.memory;
                p_mb[c] = t.mb;
            }
            ++c;
        }
    }
    *n_pieces = c;
    *m_unit = out.m_unit;
    return QRM_OK;
}

QRM_EXPORT qrm_status qrm_warmup_profile_mode(qrm_ctx* c, const uint8_t* images, int64_t count, int w, int h,
                                              int64_t stride, int iters, int b0, int mode, double* time,
                                              double* memory) {
    // warmup_profile (sim.cpp:240-288) for the device stages: medians of
    // cudaEvent-timed runs of transfer / decode / correct+return at batch b0,
    // with the transfer of host-pipeline mode `mode` (0: zero-copy window
    // fetch, 1: full-image copy).
    qrm_status s = check_uniform(c, images, count, w, h, stride);
    if (s != QRM_OK) return s;
    if (iters < 1) return fail(QRM_INVALID_INPUT, "need at least one warm-up iteration");
    if (count == 0) return fail(QRM_INVALID_INPUT, "warm-up needs at least one image");
    if (mode != 0 && mode != 1) return fail(QRM_INVALID_INPUT, "warm-up mode must be 0 (window fetch) or 1 (full image)");
    if ((s = set_device(c->device)) != QRM_OK) return s;
    b0 = static_cast<int>(std::min<int64_t>(std::max(1, b0), count));
    const int64_t img_bytes = static_cast<int64_t>(w) * h * 3;
    Workspace& W = c->ws[0];
    if ((s = ensure(W.images, W.images_cap, b0 * img_bytes)) != QRM_OK) return s;
    if ((s = ensure(W.stage, W.stage_cap, static_cast<int64_t>(b0) * c->K)) != QRM_OK) return s;
    if ((s = ensure(c->d_records, c->records_cap, b0)) != QRM_OK) return s;
    int up, sw, sh, xo, yo;
    geometry(w, h, up, sw, sh, xo, yo);
    const uint8_t* mapped = nullptr;
    bool reg = false;
    cudaEvent_t a = nullptr, b = nullptr;
    auto cleanup = on_exit([&] {
        cudaDeviceSynchronize();  // nothing of this call may still read the caller's buffer
        if (a) cudaEventDestroy(a);
        if (b) cudaEventDestroy(b);
        if (reg) cudaHostUnregister(const_cast<uint8_t*>(images));
    });
    if (mode == 0) {
        cudaPointerAttributes attr{};
        if (cudaPointerGetAttributes(&attr, images) != cudaSuccess || attr.type != cudaMemoryTypeHost) {
            cudaGetLastError();
            QRM_CUDA(cudaHostRegister(const_cast<uint8_t*>(images), (b0 - 1) * stride + img_bytes,
                                      cudaHostRegisterMapped | cudaHostRegisterReadOnly));
            reg = true;
        }
        QRM_CUDA(cudaHostGetDevicePointer(reinterpret_cast<void**>(const_cast<uint8_t**>(&mapped)),
                                          const_cast<uint8_t*>(images), 0));
        if (!direct_ok(c, mapped, w, h, stride) || (3 * c->l) % 16 != 0)
            return fail(QRM_INVALID_INPUT, "window fetch needs 16-B aligned windows (use mode 1)");
    }
    std::vector<qrm_record> host(b0);
    cudaStream_t st = nullptr;
    QRM_CUDA(cudaEventCreate(&a));
    QRM_CUDA(cudaEventCreate(&b));
    auto timed = [&](auto&& body) -> double {
        cudaEventRecord(a, st);
        body();
        cudaEventRecord(b, st);
        cudaEventSynchronize(b);
        float ms = 0.f;
        cudaEventElapsedTime(&ms, a, b);
        return ms;
    };
    WindowSource hs{};
    hs.base = mapped;
    hs.image_stride = stride;
    hs.pitch = w * 3;
    hs.x_off = xo;
    hs.y_off = yo;
    hs.direct = 1;
    hs.l = c->l;
    hs.strategy = c->cfg.tile_strategy;
    hs.tile_seed = c->cfg.tile_seed;
    WindowSource staged = hs;
    staged.base = W.stage;
    staged.image_stride = c->K;
    staged.pitch = 3 * c->l;
    staged.direct = 0;
    std::vector<double> t0v, t1v, t2v;
    for (int i = 0; i < iters; ++i) {
        if (mode == 0) {
            t0v.push_back(timed([&] { fetch_stage(c, hs, w, h, b0, W.stage, st); }));
            t1v.push_back(timed([&] { run_detect(c, W, staged, b0, c->d_records, nullptr, nullptr, st); }));
        } else {
            t0v.push_back(timed([&] {
                cudaMemcpy2DAsync(W.images, img_bytes, images, stride, img_bytes, b0, cudaMemcpyHostToDevice, st);
            }));
            t1v.push_back(timed([&] {
                detect_uniform(c, W, W.images, b0, w, h, img_bytes, 0, c->d_records, nullptr, nullptr, st);
            }));
        }
        t2v.push_back(timed([&] {
            cudaMemcpyAsync(host.data(), c->d_records, sizeof(qrm_record) * b0, cudaMemcpyDeviceToHost, st);
        }));
    }
    auto med = [](std::vector<double> v) {
        std::sort(v.begin(), v.end());
        double x = v[v.size() / 2];
        if (v.size() % 2 == 0) x = 0.5 * (x + v[v.size() / 2 - 1]);
        return std::max(x, 1e-6);
    };
    time[0] = med(t0v);
    time[1] = med(t1v);
    time[2] = med(t2v);
    c->decode_ms_per_image = time[1] / b0;
    memory[0] = static_cast<double>(mode == 0 ? c->K : img_bytes);
    memory[1] = static_cast<double>(c->K + sizeof(PendingEntry));
    memory[2] = static_cast<double>(sizeof(qrm_record));
    QRM_CUDA(cudaGetLastError());
    return QRM_OK;
}

// GPU-aware warm-up (an extension of warmup_profile, not in the reference):
// each device stage of the mode-0 pipeline (zero-copy window fetch, decode,
// record D2H) run on s = 1, 2, 4 streams at once, each stream b0 images of its
// own; sat[k] = the best measured speedup s * T(1) / T(s). A transfer stage
// bound by the PCIe link shows ~1, a decode of a small mini-batch that leaves
// SMs idle shows up to s. time[]/memory[] as qrm_warmup_profile_mode (s = 1).
QRM_EXPORT qrm_status qrm_warmup_saturation(qrm_ctx* c, const uint8_t* images, int64_t count, int w, int h,
                                            int64_t stride, int iters, int b0, double* time, double* memory,
                                            double* sat) {
    qrm_status s = check_uniform(c, images, count, w, h, stride);
    if (s != QRM_OK) return s;
    if (iters < 1) return fail(QRM_INVALID_INPUT, "need at least one warm-up iteration");
    constexpr int kMaxS = 4;
    if (count < static_cast<int64_t>(kMaxS) * std::max(1, b0))
        return fail(QRM_INVALID_INPUT, "saturation warm-up needs 4 * b0 images");
    if ((s = set_device(c->device)) != QRM_OK) return s;
    b0 = std::max(1, b0);
    const int64_t img_bytes = static_cast<int64_t>(w) * h * 3;
    int up, sw, sh, xo, yo;
    geometry(w, h, up, sw, sh, xo, yo);
    const int64_t span_bytes = (kMaxS * static_cast<int64_t>(b0) - 1) * stride + img_bytes;
    const uint8_t* mapped = nullptr;
    bool reg = false;
    std::vector<cudaStream_t> sts(kMaxS, nullptr);
    std::vector<cudaEvent_t> evs;
    auto cleanup = on_exit([&] {
        cudaDeviceSynchronize();
        for (auto e : evs) cudaEventDestroy(e);
        for (auto st : sts)
            if (st) cudaStreamDestroy(st);
        if (reg) cudaHostUnregister(const_cast<uint8_t*>(images));
    });
    cudaPointerAttributes attr{};
    if (cudaPointerGetAttributes(&attr, images) != cudaSuccess || attr.type != cudaMemoryTypeHost) {
        cudaGetLastError();
        QRM_CUDA(cudaHostRegister(const_cast<uint8_t*>(images), span_bytes,
                                  cudaHostRegisterMapped | cudaHostRegisterReadOnly));
        reg = true;
    }
    QRM_CUDA(cudaHostGetDevicePointer(reinterpret_cast<void**>(const_cast<uint8_t**>(&mapped)),
                                      const_cast<uint8_t*>(images), 0));
    if (!direct_ok(c, mapped, w, h, stride) || (3 * c->l) % 16 != 0)
        return fail(QRM_INVALID_INPUT, "window fetch needs 16-B aligned windows");
    for (auto& st : sts) QRM_CUDA(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
    if (static_cast<int>(c->ws.size()) < 1 + kMaxS) c->ws.resize(1 + kMaxS);
    for (int j = 0; j < kMaxS; ++j) {
        Workspace& W = c->ws[1 + j];
        if ((s = ensure(W.stage, W.stage_cap, static_cast<int64_t>(b0) * c->K)) != QRM_OK) return s;
        if ((s = workspace_reserve(W, b0)) != QRM_OK) return s;
    }
    if ((s = ensure(c->d_records, c->records_cap, kMaxS * static_cast<int64_t>(b0))) != QRM_OK) return s;
    std::vector<qrm_record> host(static_cast<size_t>(kMaxS) * b0);
    for (int i = 0; i < 2 * kMaxS + 2; ++i) {
        cudaEvent_t e;
        QRM_CUDA(cudaEventCreate(&e));
        evs.push_back(e);
    }
    auto source = [&](int j) {
        WindowSource hs{};
        hs.base = mapped + static_cast<int64_t>(j) * b0 * stride;
        hs.image_stride = stride;
        hs.pitch = w * 3;
        hs.x_off = xo;
        hs.y_off = yo;
        hs.direct = 1;
        hs.l = c->l;
        hs.strategy = c->cfg.tile_strategy;
        hs.tile_seed = c->cfg.tile_seed;
        hs.first_draw = static_cast<uint64_t>(j) * b0;
        return hs;
    };
    auto staged = [&](int j) {
        WindowSource ws = source(j);
        ws.base = c->ws[1 + j].stage;
        ws.image_stride = c->K;
        ws.pitch = 3 * c->l;
        ws.direct = 0;
        return ws;
    };
    // stage k on `ns` concurrent streams: wall time from the fork to the join (ms)
    auto run = [&](int k, int ns) -> double {
        cudaEvent_t fork = evs[0], join = evs[1];
        QRM_CUDA(cudaEventRecord(fork, sts[0]));
        for (int j = 1; j < ns; ++j) QRM_CUDA(cudaStreamWaitEvent(sts[j], fork, 0));
        for (int j = 0; j < ns; ++j) {
            cudaStream_t st = sts[j];
            if (k == 0) {
                if (fetch_stage(c, source(j), w, h, b0, c->ws[1 + j].stage, st) != QRM_OK) return -1.0;
            } else if (k == 1) {
                if (run_detect(c, c->ws[1 + j], staged(j), b0, c->d_records + static_cast<int64_t>(j) * b0,
                               nullptr, nullptr, st, nullptr, nullptr, false) != QRM_OK)
                    return -1.0;
            } else {
                QRM_CUDA(cudaMemcpyAsync(host.data() + static_cast<size_t>(j) * b0,
                                         c->d_records + static_cast<int64_t>(j) * b0, sizeof(qrm_record) * b0,
                                         cudaMemcpyDeviceToHost, st));
            }
            if (j > 0) {
                QRM_CUDA(cudaEventRecord(evs[2 + j], st));
                QRM_CUDA(cudaStreamWaitEvent(sts[0], evs[2 + j], 0));
            }
        }
        QRM_CUDA(cudaEventRecord(join, sts[0]));
        QRM_CUDA(cudaEventSynchronize(join));
        float ms = 0.f;
        QRM_CUDA(cudaEventElapsedTime(&ms, fork, join));
        return ms;
    };
    auto med = [](std::vector<double> v) {
        std::sort(v.begin(), v.end());
        return std::max(v[v.size() / 2], 1e-6);
    };
    for (int k = 0; k < 3; ++k) {
        double t1 = 0.0, best = 1.0;
        for (int ns = 1; ns <= kMaxS; ns *= 2) {
            run(k, ns);  // untimed: first touch of buffers / lazy state
            std::vector<double> v;
            for (int i = 0; i < iters; ++i) {
                const double ms = run(k, ns);
                if (ms < 0) return fail(QRM_CUDA_ERROR, "saturation warm-up stage failed");
                v.push_back(ms);
            }
            const double t = med(v);
            if (ns == 1) t1 = t;
            else best = std::max(best, ns * t1 / t);
        }
        time[k] = t1;
        // speedups under 10 % are run-to-run noise, not concurrency: report none
        sat[k] = best < 1.10 ? 1.0 : best;
    }
    c->decode_ms_per_image = time[1] / b0;
    memory[0] = static_cast<double>(c->K);
    memory[1] = static_cast<double>(c->K + sizeof(PendingEntry));
    memory[2] = static_cast<double>(sizeof(qrm_record));
    QRM_CUDA(cudaGetLastError());
    return QRM_OK;
}

QRM_EXPORT qrm_status qrm_warmup_profile(qrm_ctx* c, const uint8_t* images, int64_t count, int w, int h,
                                         int64_t stride, int iters, int b0, double* time, double* memory) {
    return qrm_warmup_profile_mode(c, images, count, w, h, stride, iters, b0, 1, time, memory);
}

}  // extern "C"
