// api.cu -- the C ABI (include/smlm.h): adapter pools, validation, plan staging, dispatch.
//
// PAPER.md mapping:
//   * per-(layer, projection) pool, adapters loaded/unloaded at runtime
//   * shared base weight passed per call, never copied ("no additional GPU memory overhead")
//   * static slot scale x dynamic per-request scale
//   * backward for fine-tune rows only, gradients masked per adapter
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>
#include <math.h>
#include <stdlib.h>
#include <string.h>

#include <algorithm>
#include <atomic>
#include <mutex>
#include <string>
#include <vector>

#include "../../include/smlm.h"
#include "device_types.h"
#include "plan.h"

namespace smlm {
int gemm_stages(int r_pad, size_t *smem_bytes);
int launch_gemm(const GemmArgs &a, bool bwd, int num_sms, cudaStream_t st);
int gemm2_stages(int r_pad);
int launch_gemm2(const Gemm2Args &a, bool bwd, int num_sms, cudaStream_t st);
int launch_u(const UArgs &a, int num_sms, cudaStream_t st);
int launch_shrink_short(const __nv_bfloat16 *X, const SlotDev *slots, const DevBlock *blocks,
                        const DevShortRow *srows, int n_blocks, int in_f, int r, int r_pad, __nv_bfloat16 *Vbd,
                        __nv_bfloat16 *Vsave, cudaStream_t st);
template <typename T>
int launch_rows_shrink(const DevTile *tiles, int n_tiles, const SlotDev *slots, const T *X, int in_f, int r,
                       float *Vf, T *Vsave, int ft_only, cudaStream_t st);
template <typename T>
int launch_rows_u(const DevTile *tiles, int n_tiles, const SlotDev *slots, const T *dY, int out_f, int r, float *Uf,
                  __nv_bfloat16 *sUt, int r_pad, cudaStream_t st);
template <typename TV>
int launch_prep_sv(const DevTile *tiles, int n_tiles, const TV *V, int r, int r_pad, __nv_bfloat16 *sVt,
                   cudaStream_t st);
int launch_tok(const TokArgs &a, int num_sms, cudaStream_t st);
int dec_stages();
int dec_chunks(int in_f);
int launch_shrink_split(const __nv_bfloat16 *X, const SlotDev *slots, const DevBlock *blocks,
                        const DevShortRow *srows, int n_blocks, int in_f, int r, int r_pad, float *part,
                        __nv_bfloat16 *Vbd, __nv_bfloat16 *Vsave, cudaStream_t st);
int launch_dec(const DecArgs &a, int num_sms, cudaStream_t st);
int launch_decf(const DecFArgs &a, cudaStream_t st);
size_t grad_group_bytes();
void fill_grad_group(void *dst, int slot, int tile_begin, int n_tiles, float *dA, float *dB);
template <typename T, typename TV>
int launch_dadb(const DevTile *tiles, const void *groups, int n_groups, const T *X, const T *dY, const float *Uf,
                const TV *V, int in_f, int out_f, int r, int accumulate, cudaStream_t st);
int launch_f32_fwd(const DevTile *tiles, int n_tiles, const SlotDev *slots, const float *X, const float *W, float *Y,
                   const float *Vf, int in_f, int out_f, int r, cudaStream_t st);
int launch_f32_dx(const DevTile *tiles, int n_tiles, const SlotDev *slots, const float *dY, const float *W, float *dX,
                  const float *Uf, int in_f, int out_f, int r, cudaStream_t st);
}  // namespace smlm

using namespace smlm;

// ------------------------------------------------------------------------------------------
// error reporting, instrumentation
// ------------------------------------------------------------------------------------------
static thread_local std::string g_last_error;
static std::atomic<uint64_t> g_launches{0};

static int set_err(int code, const std::string &msg) {
    g_last_error = msg;
    return code;
}
static int cuda_err(cudaError_t e, const char *where) {
    return set_err(SMLM_E_CUDA, std::string(where) + ": " + cudaGetErrorString(e));
}
#define CK(call)                                                   \
    do {                                                           \
        cudaError_t _e = (call);                                   \
        if (_e != cudaSuccess) return cuda_err(_e, #call);         \
    } while (0)
#define CKL(expr, n)                                               \
    do {                                                           \
        int _e = (expr);                                           \
        if (_e != 0) return cuda_err((cudaError_t)_e, #expr);      \
        g_launches += (n);                                         \
    } while (0)

namespace {

struct Profiler {
    std::mutex mu;
    int mask = 0;   // bit k: record kernel class k
    struct Rec { cudaEvent_t a, b; int kind; };
    std::vector<Rec> recs;
    std::vector<cudaEvent_t> pool;
    cudaEvent_t get() {
        if (!pool.empty()) { cudaEvent_t e = pool.back(); pool.pop_back(); return e; }
        cudaEvent_t e;
        cudaEventCreate(&e);
        return e;
    }
} g_prof;

struct ProfScope {
    cudaEvent_t a = nullptr;
    int kind;
    cudaStream_t st;
    ProfScope(int k, cudaStream_t s) : kind(k), st(s) {
        if (g_prof.mask & (1 << k)) {
            std::lock_guard<std::mutex> lk(g_prof.mu);
            a = g_prof.get();
            cudaEventRecord(a, st);
        }
    }
    ~ProfScope() {
        if (a) {
            std::lock_guard<std::mutex> lk(g_prof.mu);
            cudaEvent_t b = g_prof.get();
            cudaEventRecord(b, st);
            g_prof.recs.push_back({a, b, kind});
        }
    }
};

// ------------------------------------------------------------------------------------------
// TMA descriptor encoding through the driver entry point (no -lcuda link dependency)
// ------------------------------------------------------------------------------------------
PFN_cuTensorMapEncodeTiled_v12000 g_encode = nullptr;

int get_encode() {
    if (g_encode) return SMLM_OK;
    void *fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    cudaError_t e = cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
    if (e != cudaSuccess || !fn) return set_err(SMLM_E_CUDA, "cuTensorMapEncodeTiled entry point unavailable");
    g_encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
    return SMLM_OK;
}

CUtensorMapSwizzle swizzle_for(int row_bytes) {
    return row_bytes >= 128 ? CU_TENSOR_MAP_SWIZZLE_128B
                            : (row_bytes == 64 ? CU_TENSOR_MAP_SWIZZLE_64B : CU_TENSOR_MAP_SWIZZLE_32B);
}

// 2-D bf16 tensor [outer, inner] row-major
int make_map(CUtensorMap *m, const void *ptr, uint64_t inner, uint64_t outer, uint32_t box_inner,
             uint32_t box_outer, CUtensorMapSwizzle swz) {
    if (get_encode() != SMLM_OK) return SMLM_E_CUDA;
    cuuint64_t dims[2] = {inner, outer};
    cuuint64_t strides[1] = {inner * 2};
    cuuint32_t box[2] = {box_inner, box_outer};
    cuuint32_t es[2] = {1, 1};
    CUresult r = g_encode(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void *>(ptr), dims, strides, box, es,
                          CU_TENSOR_MAP_INTERLEAVE_NONE, swz, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                          CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) return set_err(SMLM_E_CUDA, "cuTensorMapEncodeTiled failed (" + std::to_string((int)r) + ")");
    return SMLM_OK;
}

// ------------------------------------------------------------------------------------------
// pinned staging ring (plan uploads and slot-table updates stay stream-ordered, no host sync)
// ------------------------------------------------------------------------------------------
struct Ring {
    struct Ent {
        void *host = nullptr;
        size_t cap = 0;
        cudaEvent_t ev = nullptr;
        bool pending = false;
    };
    Ent e[8];
    int next = 0;
    ~Ring() {
        for (auto &x : e) {
            if (x.pending) cudaEventSynchronize(x.ev);
            if (x.host) cudaFreeHost(x.host);
            if (x.ev) cudaEventDestroy(x.ev);
        }
    }
    // returns index of a free pinned buffer with >= bytes capacity
    int acquire(size_t bytes, void **host) {
        Ent &x = e[next];
        if (x.pending) {
            cudaEventSynchronize(x.ev);
            x.pending = false;
        }
        if (x.cap < bytes) {
            if (x.host) cudaFreeHost(x.host);
            x.host = nullptr;
            size_t cap = bytes < 65536 ? 65536 : bytes * 2;
            if (cudaMallocHost(&x.host, cap) != cudaSuccess) return -1;
            x.cap = cap;
        }
        if (!x.ev) cudaEventCreateWithFlags(&x.ev, cudaEventDisableTiming);
        *host = x.host;
        int idx = next;
        next = (next + 1) % 8;
        return idx;
    }
    void release(int idx, cudaStream_t st) {
        cudaEventRecord(e[idx].ev, st);
        e[idx].pending = true;
    }
};

struct SlotHost {
    bool used = false;
    const void *A = nullptr;
    const void *B = nullptr;
    float scale = 1.f;
    float *dA = nullptr;
    float *dB = nullptr;
};

size_t align256(size_t x) { return (x + 255) & ~size_t(255); }

// m-tiles per raster group: the group's 128-row A tiles (128 x K bf16) stay L2-resident while
// the CTAs sweep every n-tile, so each W n-tile is fetched from HBM once per group (~48 MB budget)
int raster_group(int K) {
    const long tile = 128L * K * 2;
    long g = (48L << 20) / tile;
    if (g < 4) g = 4;
    if (g > 64) g = 64;
    return (int)g;
}

}  // namespace

struct smlm_pool_s {
    int device = 0;
    int in = 0, out = 0, r = 0, r_pad = 16, cap = 0, dtype = 0;
    int l_long = 64;
    int cta_pair = 1;   // forward long tiles on CTA pairs (cta_group::2)
    int num_sms = 148;
    std::vector<SlotHost> slots;
    std::vector<uint8_t> ok;
    std::vector<float> scales;
    SlotDev *d_slots = nullptr;
    unsigned long long *d_counter = nullptr;   // fused decode kernel: release counter
    unsigned long long dec_epoch = 0;
    Ring ring;
};

namespace {

struct DeviceGuard {
    int prev = -1;
    explicit DeviceGuard(int dev) {
        cudaGetDevice(&prev);
        if (prev != dev) cudaSetDevice(dev);
    }
    ~DeviceGuard() {
        int cur;
        cudaGetDevice(&cur);
        if (prev >= 0 && cur != prev) cudaSetDevice(prev);
    }
};

int check_sticky() {
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return cuda_err(e, "pending CUDA error");
    return SMLM_OK;
}

// Sizes of the workspace sections for a planned call.
struct WsLayout {
    size_t plan_off = 0, plan_bytes = 0;
    size_t vbd_off = 0, vbd_bytes = 0;     // bf16 fwd: block-diagonal s*V of short tiles
    size_t u_off = 0, u_bytes = 0;         // bwd fp32 mode: U fp32 [S,r]
    size_t sut_off = 0, svt_off = 0, st_bytes = 0;  // bwd bf16: tile-compact s*U, s*V [tiles*128, r_pad]
    size_t upart_off = 0, upart_bytes = 0; // bwd bf16: split-K partials of U = dY B_a
    int u_items = 0, u_ksplit = 0;
    size_t vf_off = 0, vf_bytes = 0;       // fp32 V [S,r] (fp32 mode, or bwd recompute)
    size_t spart_off = 0, spart_bytes = 0; // bf16 fwd: K-split shrink partials
    size_t dpart_off = 0, dpart_bytes = 0; // bf16 fwd decode GEMM: split-K partials
    int dec_items = 0, dec_ksplit = 0;     // > 0: pure-decode batch takes the transposed split-K kernel
    int dec_cmc = 1;
    std::vector<int> dec_uniq;             // distinct adapter slots of the decode batch
    bool decf = false;                     // fused single-launch decode kernel
    int decf_ksplit = 0;
    size_t vg_off = 0;
    size_t total = 0;
};

int plan_for(smlm_pool p, const smlm_batch *b, bool bwd, Plan &plan) {
    std::string msg;
    // fp32 test mode consumes segment-aligned tiles for every row (L_long = 1)
    int l_long = p->dtype == SMLM_FP32 ? 1 : p->l_long;
    int rc = build_plan(b, p->cap, p->ok.data(), p->scales.data(), l_long, bwd, plan, msg);
    if (rc != SMLM_OK) return set_err(rc, msg);
    return SMLM_OK;
}

WsLayout layout_for(smlm_pool p, const smlm_batch *b, const Plan &plan, bool bwd, bool need_vf) {
    WsLayout L;
    size_t off = 0;
    if (!bwd) {
        L.plan_bytes = (plan.long_tiles.size() + plan.short_tiles.size()) * sizeof(DevTile) +
                       plan.blocks.size() * sizeof(DevBlock) + plan.short_rows.size() * sizeof(DevShortRow) +
                       // decode-path extras: distinct slots + per-row records (<= 4 short tiles)
                       (size_t)p->cap * 4 + 4 * 128 * sizeof(DecRow) + 64 +
                       (plan.long_tiles.size() + plan.short_tiles.size()) * sizeof(DevPair) + 16;
    } else {
        L.plan_bytes = plan.bwd_tiles.size() * (sizeof(DevTile) + 4 + sizeof(DevPair)) +
                       plan.groups.size() * grad_group_bytes() + 64;
    }
    L.plan_off = off;
    off = align256(off + L.plan_bytes + 16);
    if (!bwd && p->dtype == SMLM_BF16) {
        L.vbd_off = off;
        L.vbd_bytes = plan.blocks.size() * 128 * (size_t)p->r_pad * 2;
        off = align256(off + L.vbd_bytes);
        const int nch = dec_chunks(p->in);
        if (nch > 0) {
            L.spart_off = off;
            L.spart_bytes = plan.blocks.size() * (size_t)nch * 128 * p->r_pad * 4;
            off = align256(off + L.spart_bytes);
        }
        // pure decode / short batches (<= 512 rows in <= 4 short tiles): transposed split-K GEMM
        const int nst = (int)plan.short_tiles.size();
        if (plan.long_tiles.empty() && nst > 0 && nst <= 4) {
            std::vector<int> uniq;
            for (auto &bk : plan.blocks) uniq.push_back(bk.slot);
            std::sort(uniq.begin(), uniq.end());
            uniq.erase(std::unique(uniq.begin(), uniq.end()), uniq.end());
            const int groups = (nst + 1) / 2;
            const int n_nt = (p->out + 127) / 128;
            const int n_vt = ((int)uniq.size() * p->r_pad + 127) / 128;
            // opt-in (SMLM_DEC_MC=1): clusters of 4 row tiles share the X tile by TMA multicast;
            // measured slower (the 4 CTAs must all release a stage before it is refilled)
            const int cmc = getenv("SMLM_DEC_MC") ? 4 : 1;
            L.dec_cmc = cmc;
            const int items = ((n_nt + n_vt + cmc - 1) / cmc) * cmc * groups;
            int ks = p->num_sms / items;        // one wave
            if (const char *e = getenv("SMLM_DEC_KSPLIT")) ks = atoi(e);   // measurement override
            const int nkb = p->in / 64;
            const int ks_bytes = p->in / 256;   // partials <= ~2x the W bytes
            if (ks > ks_bytes) ks = ks_bytes;
            if (ks > nkb / 2) ks = nkb / 2;
            if (ks < 1) ks = 1;
            L.dec_items = items;
            L.dec_ksplit = ks;
            L.dec_uniq = uniq;
            // <= 256 decode rows: fused single-launch kernel (DSMEM split-K reduction, in-kernel expand)
            // experimental (opt-in, SMLM_DECF=1): measured slower than the two-kernel path so far
            if (nst <= 2 && getenv("SMLM_DECF")) {
                const int tiles_f = n_nt + n_vt;
                const int m_rows = 128 * nst;
                // power-of-two cluster <= 8 (portable): every cluster of a GPC-sized group co-resides
                int kf = 1;
                while (kf * 2 <= 8 && tiles_f * kf * 2 <= p->num_sms) kf *= 2;
                if (const char *e = getenv("SMLM_DECF_KSPLIT")) kf = atoi(e);
                if (kf > nkb) kf = nkb;
                if (kf * 64 < m_rows) kf = (m_rows + 63) / 64;   // <= 64 decode rows per CTA slice
                if (kf <= 8 && kf <= nkb && tiles_f * kf <= p->num_sms) {
                    L.decf = true;
                    L.decf_ksplit = kf;
                }
            }
            if (L.decf) {
                L.vg_off = off;
                off = align256(off + 256 * (size_t)p->r_pad * 4);
            } else {
                L.dpart_off = off;
                L.dpart_bytes = (size_t)items * ks * 256 * 128 * 4;
                off = align256(off + L.dpart_bytes);
            }
        }
    }
    if (bwd && p->dtype == SMLM_FP32) {
        L.u_off = off;
        L.u_bytes = (size_t)b->S * p->r * 4;
        off = align256(off + L.u_bytes);
    }
    if (bwd && p->dtype == SMLM_BF16) {
        L.st_bytes = plan.bwd_tiles.size() * 128 * (size_t)p->r_pad * 2;
        L.sut_off = off;
        off = align256(off + L.st_bytes);
        L.svt_off = off;
        off = align256(off + L.st_bytes);
        for (auto &t : plan.bwd_tiles)
            if (t.slot >= 0) ++L.u_items;
        if (L.u_items) {
            int ks = p->num_sms / L.u_items;
            const int nkb = p->out / 64;
            if (ks > nkb / 4) ks = nkb / 4;
            if (ks < 1) ks = 1;
            L.u_ksplit = ks;
            L.upart_off = off;
            L.upart_bytes = (size_t)L.u_items * ks * 128 * p->r_pad * 4;
            off = align256(off + L.upart_bytes);
        }
    }
    if (need_vf) {
        L.vf_off = off;
        L.vf_bytes = (size_t)b->S * p->r * 4;
        off = align256(off + L.vf_bytes);
    }
    L.total = off;
    return L;
}

// Copy a host byte vector into the workspace through the pinned ring (stream ordered).
int stage_upload(smlm_pool p, const std::vector<uint8_t> &bytes, void *dst, cudaStream_t st) {
    if (bytes.empty()) return SMLM_OK;
    void *h = nullptr;
    int idx = p->ring.acquire(bytes.size(), &h);
    if (idx < 0) return set_err(SMLM_E_CUDA, "cudaMallocHost failed");
    memcpy(h, bytes.data(), bytes.size());
    cudaError_t e = cudaMemcpyAsync(dst, h, bytes.size(), cudaMemcpyHostToDevice, st);
    p->ring.release(idx, st);
    if (e != cudaSuccess) return cuda_err(e, "plan upload");
    return SMLM_OK;
}

template <typename T> void append(std::vector<uint8_t> &v, const std::vector<T> &x) {
    const uint8_t *s = reinterpret_cast<const uint8_t *>(x.data());
    v.insert(v.end(), s, s + x.size() * sizeof(T));
}

}  // namespace

// ==========================================================================================
// C ABI
// ==========================================================================================
extern "C" {

const char *smlm_status_string(int s) {
    switch (s) {
        case SMLM_OK: return "SMLM_OK";
        case SMLM_E_INVALID: return "SMLM_E_INVALID";
        case SMLM_E_SHAPE: return "SMLM_E_SHAPE";
        case SMLM_E_SLOT: return "SMLM_E_SLOT";
        case SMLM_E_CAPACITY: return "SMLM_E_CAPACITY";
        case SMLM_E_CUDA: return "SMLM_E_CUDA";
        case SMLM_E_UNSUPPORTED: return "SMLM_E_UNSUPPORTED";
        case SMLM_E_WORKSPACE: return "SMLM_E_WORKSPACE";
    }
    return "SMLM_E_UNKNOWN";
}

const char *smlm_last_error(void) { return g_last_error.c_str(); }

uint64_t smlm_launch_count(void) { return g_launches.load(); }

int smlm_profile_enable(int on) {
    std::lock_guard<std::mutex> lk(g_prof.mu);
    g_prof.mask = on;
    return SMLM_OK;
}

int smlm_profile_read(int kind, double *total_ms, int *count) {
    std::lock_guard<std::mutex> lk(g_prof.mu);
    double tot = 0;
    int n = 0;
    std::vector<Profiler::Rec> keep;
    for (auto &r : g_prof.recs) {
        if (r.kind != kind) { keep.push_back(r); continue; }
        cudaEventSynchronize(r.b);
        float ms = 0;
        cudaEventElapsedTime(&ms, r.a, r.b);
        tot += ms;
        ++n;
        g_prof.pool.push_back(r.a);
        g_prof.pool.push_back(r.b);
    }
    g_prof.recs.swap(keep);
    if (total_ms) *total_ms = tot;
    if (count) *count = n;
    return SMLM_OK;
}

int smlm_pool_create(int device, int in_features, int out_features, int rank, int capacity, int dtype,
                     smlm_pool *out) {
    if (!out) return set_err(SMLM_E_INVALID, "out is NULL");
    *out = nullptr;
    if (capacity < 1) return set_err(SMLM_E_INVALID, "capacity must be >= 1");
    if (in_features < 1 || out_features < 1 || rank < 1) return set_err(SMLM_E_INVALID, "bad shape");
    if (dtype == SMLM_BF16) {
        if (!(rank == 8 || rank == 16 || rank == 32 || rank == 64))
            return set_err(SMLM_E_UNSUPPORTED, "bf16 path supports rank in {8,16,32,64}");
        if (in_features % 64 || out_features % 64)
            return set_err(SMLM_E_UNSUPPORTED, "bf16 path needs in/out multiples of 64");
    } else if (dtype == SMLM_FP32) {
        if (rank > 64) return set_err(SMLM_E_UNSUPPORTED, "fp32 path supports rank <= 64");
    } else {
        return set_err(SMLM_E_INVALID, "unknown dtype");
    }
    int ndev = 0;
    cudaError_t e = cudaGetDeviceCount(&ndev);
    if (e != cudaSuccess || device < 0 || device >= ndev)
        return set_err(SMLM_E_UNSUPPORTED, "no such CUDA device (there is no CPU fallback)");
    cudaDeviceProp prop;
    CK(cudaGetDeviceProperties(&prop, device));
    if (prop.major != 10 || prop.minor != 0)
        return set_err(SMLM_E_UNSUPPORTED, "device is not sm_100 (B200); this library is sm_100a-only");
    DeviceGuard dg(device);
    auto *p = new smlm_pool_s();
    p->device = device;
    p->in = in_features;
    p->out = out_features;
    p->r = rank;
    p->r_pad = rank <= 16 ? 16 : (rank <= 32 ? 32 : 64);
    p->cap = capacity;
    p->dtype = dtype;
    p->num_sms = prop.multiProcessorCount;
    p->slots.resize(capacity);
    p->ok.assign(capacity, 0);
    p->scales.assign(capacity, 0.f);
    e = cudaMalloc(&p->d_slots, sizeof(SlotDev) * capacity);
    if (e != cudaSuccess) {
        delete p;
        return cuda_err(e, "cudaMalloc(slot table)");
    }
    if (e == cudaSuccess) e = cudaMalloc(&p->d_counter, 64);
    if (e == cudaSuccess) e = cudaMemset(p->d_counter, 0, 64);
    if (e == cudaSuccess) e = cudaMemset(p->d_slots, 0, sizeof(SlotDev) * capacity);
    if (e != cudaSuccess) {
        cudaFree(p->d_slots);
        delete p;
        return cuda_err(e, "cudaMemset(slot table)");
    }
    *out = p;
    return SMLM_OK;
}

int smlm_pool_destroy(smlm_pool p) {
    if (!p) return SMLM_OK;
    {
        DeviceGuard dg(p->device);
        cudaDeviceSynchronize();
        if (p->d_slots) cudaFree(p->d_slots);
        if (p->d_counter) cudaFree(p->d_counter);
    }
    delete p;
    return SMLM_OK;
}

int smlm_pool_set_option(smlm_pool p, int option, int value) {
    if (!p) return set_err(SMLM_E_INVALID, "pool is NULL");
    if (option == SMLM_OPT_L_LONG) {
        if (value < 1) return set_err(SMLM_E_INVALID, "L_long must be >= 1");
        p->l_long = value;
        return SMLM_OK;
    }
    if (option == SMLM_OPT_CTA_PAIR) {
        p->cta_pair = value != 0;
        return SMLM_OK;
    }
    return set_err(SMLM_E_INVALID, "unknown option");
}

static int upload_slot(smlm_pool p, int slot, cudaStream_t st) {
    SlotDev d;
    memset(&d, 0, sizeof(d));
    const SlotHost &h = p->slots[slot];
    if (h.used) {
        d.A = h.A;
        d.B = h.B;
        d.dA = h.dA;
        d.dB = h.dB;
        d.scale = h.scale;
        d.used = 1;
        if (p->dtype == SMLM_BF16) {
            const int rb = p->r_pad * 2;
            int rc;
            if ((rc = make_map(&d.tmA, h.A, p->in, p->r, 64, p->r_pad, CU_TENSOR_MAP_SWIZZLE_128B))) return rc;
            // forward n-tile = 256 - r_pad output columns (the shrink rides in the same N=256 MMA)
            if ((rc = make_map(&d.tmBn, h.B, p->r, p->out, p->r_pad, 256 - p->r_pad, swizzle_for(rb)))) return rc;
            if ((rc = make_map(&d.tmBk, h.B, p->r, p->out, p->r_pad, 64, swizzle_for(rb)))) return rc;
        }
    }
    std::vector<uint8_t> bytes(sizeof(SlotDev));
    memcpy(bytes.data(), &d, sizeof(SlotDev));
    return stage_upload(p, bytes, p->d_slots + slot, st);
}

int smlm_adapter_register(smlm_pool p, const void *A, const void *B, float scale, void *stream, int *slot_out) {
    if (!p || !A || !B || !slot_out) return set_err(SMLM_E_INVALID, "NULL argument");
    if (!(scale > 0.f) || !isfinite(scale)) return set_err(SMLM_E_INVALID, "scale must be finite and > 0");
    if (p->dtype == SMLM_BF16 && (((uintptr_t)A & 15) || ((uintptr_t)B & 15)))
        return set_err(SMLM_E_INVALID, "A/B must be 16-byte aligned");
    int slot = -1;
    for (int i = 0; i < p->cap; ++i)
        if (!p->slots[i].used) { slot = i; break; }
    if (slot < 0) return set_err(SMLM_E_CAPACITY, "adapter pool is full");
    DeviceGuard dg(p->device);
    int rc = check_sticky();
    if (rc) return rc;
    SlotHost &h = p->slots[slot];
    h.used = true;
    h.A = A;
    h.B = B;
    h.scale = scale;
    h.dA = h.dB = nullptr;
    rc = upload_slot(p, slot, (cudaStream_t)stream);
    if (rc) {
        h = SlotHost();
        return rc;
    }
    p->ok[slot] = 1;
    p->scales[slot] = scale;
    *slot_out = slot;
    return SMLM_OK;
}

int smlm_adapter_set_grad(smlm_pool p, int slot, float *dA, float *dB) {
    if (!p) return set_err(SMLM_E_INVALID, "pool is NULL");
    if (slot < 0 || slot >= p->cap || !p->slots[slot].used) return set_err(SMLM_E_SLOT, "slot not registered");
    p->slots[slot].dA = dA;
    p->slots[slot].dB = dB;
    return SMLM_OK;
}

int smlm_adapter_unregister(smlm_pool p, int slot, void *stream) {
    if (!p) return set_err(SMLM_E_INVALID, "pool is NULL");
    if (slot < 0 || slot >= p->cap || !p->slots[slot].used) return set_err(SMLM_E_SLOT, "slot not registered");
    DeviceGuard dg(p->device);
    p->slots[slot] = SlotHost();
    p->ok[slot] = 0;
    p->scales[slot] = 0.f;
    return upload_slot(p, slot, (cudaStream_t)stream);
}

int smlm_plan(const smlm_batch *batch, int capacity, const uint8_t *slot_registered, int l_long, int backward,
              int32_t *items, int max_items, int *n_items) {
    if (!n_items) return set_err(SMLM_E_INVALID, "n_items is NULL");
    Plan plan;
    std::string msg;
    int rc = build_plan(batch, capacity, slot_registered, nullptr, l_long, backward != 0, plan, msg);
    if (rc) return set_err(rc, msg);
    std::vector<int32_t> rec;
    export_plan(plan, batch, backward != 0, rec);
    int n = (int)(rec.size() / 6);
    *n_items = n;
    if (n > max_items || (n > 0 && !items)) return set_err(SMLM_E_WORKSPACE, "items buffer too small");
    if (n) memcpy(items, rec.data(), rec.size() * sizeof(int32_t));
    return SMLM_OK;
}

int smlm_plan_export(smlm_pool p, const smlm_batch *batch, int backward, int32_t *items, int max_items,
                     int *n_items) {
    if (!p) return set_err(SMLM_E_INVALID, "pool is NULL");
    return smlm_plan(batch, p->cap, p->ok.data(), p->l_long, backward, items, max_items, n_items);
}

size_t smlm_workspace_size(smlm_pool p, const smlm_batch *batch, int backward) {
    if (!p) return 0;
    Plan plan;
    if (plan_for(p, batch, backward != 0, plan) != SMLM_OK) return 0;
    bool need_vf = p->dtype == SMLM_FP32 || backward;  // conservative: bwd may recompute V (V_save NULL)
    return layout_for(p, batch, plan, backward != 0, need_vf).total;
}

int smlm_forward(smlm_pool p, const smlm_batch *b, const void *X, const void *W, void *Y, void *V_save, void *ws,
                 size_t ws_bytes, void *stream) {
    if (!p || !b) return set_err(SMLM_E_INVALID, "NULL pool/batch");
    Plan plan;
    int rc = plan_for(p, b, false, plan);
    if (rc) return rc;
    if (b->S == 0 || b->G == 0) return SMLM_OK;
    if (!X || !Y) return set_err(SMLM_E_INVALID, "X and Y must be non-NULL");
    const bool need_vf = p->dtype == SMLM_FP32;
    WsLayout L = layout_for(p, b, plan, false, need_vf);
    if (!ws || ws_bytes < L.total) return set_err(SMLM_E_WORKSPACE, "workspace too small");
    DeviceGuard dg(p->device);
    if ((rc = check_sticky())) return rc;
    cudaStream_t st = (cudaStream_t)stream;
    uint8_t *wsb = reinterpret_cast<uint8_t *>(ws);

    if (p->dtype == SMLM_FP32) {
        std::vector<uint8_t> bytes;
        append(bytes, plan.long_tiles);
        if ((rc = stage_upload(p, bytes, wsb + L.plan_off, st))) return rc;
        const DevTile *tiles = reinterpret_cast<const DevTile *>(wsb + L.plan_off);
        const int nt = (int)plan.long_tiles.size();
        float *Vf = reinterpret_cast<float *>(wsb + L.vf_off);
        CKL(launch_rows_shrink<float>(tiles, nt, p->d_slots, (const float *)X, p->in, p->r, Vf, (float *)V_save, 1,
                                      st), 1);
        CKL(launch_f32_fwd(tiles, nt, p->d_slots, (const float *)X, (const float *)W, (float *)Y, Vf, p->in, p->out,
                           p->r, st), 1);
        return SMLM_OK;
    }

    // ---------------- bf16 tensor-core path ----------------
    const bool has_w = W != nullptr;
    std::vector<DevTile> tiles;
    tiles.reserve(plan.long_tiles.size() + plan.short_tiles.size());
    for (auto &t : plan.long_tiles)
        if (has_w || (t.flags & kTileLora)) tiles.push_back(t);
    for (auto &t : plan.short_tiles)
        if (has_w || t.nblk > 0) tiles.push_back(t);
    // pairs of long tiles (same segment) for the CTA-pair kernel
    int n_long_kept = 0;
    for (auto &t : tiles)
        if (!(t.flags & kTileShort)) ++n_long_kept;
    std::vector<DevPair> pairs;
    if (has_w && p->cta_pair) {
        for (int i = 0; i < n_long_kept;) {
            const DevTile &t0 = tiles[i];
            DevPair pr{};
            pr.row0 = t0.row0;
            pr.slot = t0.slot;
            pr.flags = (t0.flags & kTileFT) ? kPairFT : 0;
            pr.scale = t0.scale;
            int rows = t0.rows;
            if (i + 1 < n_long_kept && tiles[i + 1].seg == t0.seg) {
                rows = 128 + tiles[i + 1].rows;
                i += 2;
            } else {
                i += 1;
            }
            pr.rows = rows;
            pairs.push_back(pr);
        }
        // short tiles ride in the same launch: one per pair, CTA 1 a masked dummy
        for (size_t i = n_long_kept; i < tiles.size(); ++i) {
            const DevTile &t = tiles[i];
            DevPair pr{};
            pr.row0 = t.row0;
            pr.rows = t.rows;
            pr.slot = -1;
            pr.flags = kPairShort;
            pr.blk0 = t.blk0;
            pr.nblk = t.nblk;
            pairs.push_back(pr);
        }
    }
    std::vector<uint8_t> bytes;
    append(bytes, tiles);
    const size_t blk_off = bytes.size();
    append(bytes, plan.blocks);
    const size_t srow_off = bytes.size();
    append(bytes, plan.short_rows);
    while (bytes.size() % 16) bytes.push_back(0);
    const size_t pair_off = bytes.size();
    append(bytes, pairs);
    const DevTile *d_tiles = reinterpret_cast<const DevTile *>(wsb + L.plan_off);
    const DevBlock *d_blocks = reinterpret_cast<const DevBlock *>(wsb + L.plan_off + blk_off);
    const DevShortRow *d_srows = reinterpret_cast<const DevShortRow *>(wsb + L.plan_off + srow_off);
    __nv_bfloat16 *Vbd = reinterpret_cast<__nv_bfloat16 *>(wsb + L.vbd_off);

    if (has_w && L.dec_items > 0) {
        // pure decode batch: one streaming pass over [W ; A_u] (base rows + rank-r rows of every
        // adapter in the batch) with split K, then a wide reduce + expand pass
        const int groups = ((int)tiles.size() + 1) / 2;
        std::vector<DecRow> drows((size_t)groups * 256, DecRow{-1, -1, 0.f, 0});
        std::vector<int> uidx_of(p->cap, -1);
        for (size_t i = 0; i < L.dec_uniq.size(); ++i) uidx_of[L.dec_uniq[i]] = (int)i;
        for (size_t t = 0; t < tiles.size(); ++t) {
            const DevTile &tl = tiles[t];
            for (int m = 0; m < tl.rows; ++m) drows[t * 128 + m] = DecRow{tl.row0 + m, -1, 0.f, 0};
            for (int bi = 0; bi < tl.nblk; ++bi) {
                const DevBlock &bk = plan.blocks[tl.blk0 + bi];
                for (int i = 0; i < bk.nrows; ++i) {
                    const DevShortRow &sr = plan.short_rows[bk.row_begin + i];
                    drows[t * 128 + sr.pos] = DecRow{sr.row, uidx_of[bk.slot], sr.scale, sr.ft};
                }
            }
        }
        std::vector<uint8_t> extra;
        const size_t vt_off = bytes.size();
        append(extra, L.dec_uniq);
        while (extra.size() % 16) extra.push_back(0);
        const size_t rows_off = vt_off + extra.size();
        append(extra, drows);
        bytes.insert(bytes.end(), extra.begin(), extra.end());
        if ((rc = stage_upload(p, bytes, wsb + L.plan_off, st))) return rc;
        if (L.decf) {
            DecFArgs f;
            memset(&f, 0, sizeof(f));
            if ((rc = make_map(&f.tmW, W, p->in, p->out, 64, 128, CU_TENSOR_MAP_SWIZZLE_128B))) return rc;
            if ((rc = make_map(&f.tmX, X, p->in, b->S, 64, 128, CU_TENSOR_MAP_SWIZZLE_128B))) return rc;
            f.slots = p->d_slots;
            f.vt_slots = reinterpret_cast<const int *>(wsb + L.plan_off + vt_off);
            f.rows = reinterpret_cast<const DecRow *>(wsb + L.plan_off + rows_off);
            for (size_t t = 0; t < tiles.size() && t < 2; ++t) f.tile_row0[t] = tiles[t].row0;
            f.n_uniq = (int)L.dec_uniq.size();
            f.n_vt = (f.n_uniq * p->r_pad + 127) / 128;
            f.n_nt = (p->out + 127) / 128;
            f.ksplit = L.decf_ksplit;
            f.m_rows = 128 * (int)tiles.size();
            f.K = p->in;
            f.N = p->out;
            f.r = p->r;
            f.r_pad = p->r_pad;
            f.stages = dec_stages();
            f.Y = Y;
            f.Vsave = V_save;
            f.Vg = reinterpret_cast<float *>(wsb + L.vg_off);
            f.v_done = p->d_counter;
            p->dec_epoch += 1;
            f.v_target = p->dec_epoch * (unsigned long long)(f.n_vt * f.ksplit);
            if (f.n_vt == 0) p->dec_epoch -= 1;
            ProfScope ps(0, st);
            CKL(launch_decf(f, st), 1);
            return SMLM_OK;
        }
        DecArgs d;
        memset(&d, 0, sizeof(d));
        if ((rc = make_map(&d.tmW, W, p->in, p->out, 64, 128, CU_TENSOR_MAP_SWIZZLE_128B))) return rc;
        if ((rc = make_map(&d.tmX, X, p->in, b->S, 64, 128, CU_TENSOR_MAP_SWIZZLE_128B))) return rc;
        d.slots = p->d_slots;
        d.tiles = d_tiles;  // only short tiles (no long tiles in a pure decode batch)
        d.vt_slots = reinterpret_cast<const int *>(wsb + L.plan_off + vt_off);
        d.rows = reinterpret_cast<const DecRow *>(wsb + L.plan_off + rows_off);
        d.n_tiles = (int)tiles.size();
        d.n_groups = groups;
        d.n_nt = (p->out + 127) / 128;
        d.n_uniq = (int)L.dec_uniq.size();
        d.n_vt = (d.n_uniq * p->r_pad + 127) / 128;
        d.ksplit = L.dec_ksplit;
        d.cmc = L.dec_cmc;
        if (d.cmc > 1 && (rc = make_map(&d.tmX64, X, p->in, b->S, 64, 64, CU_TENSOR_MAP_SWIZZLE_128B))) return rc;
        d.K = p->in;
        d.N = p->out;
        d.r = p->r;
        d.r_pad = p->r_pad;
        d.stages = dec_stages();
        d.Y = Y;
        d.Vsave = V_save;
        d.part = reinterpret_cast<float *>(wsb + L.dpart_off);
        ProfScope ps(0, st);
        CKL(launch_dec(d, p->num_sms, st), 2);
        return SMLM_OK;
    }
    if ((rc = stage_upload(p, bytes, wsb + L.plan_off, st))) return rc;
    if (!plan.blocks.empty()) {
        ProfScope ps(2, st);
        if (L.spart_bytes) {
            CKL(launch_shrink_split((const __nv_bfloat16 *)X, p->d_slots, d_blocks, d_srows, (int)plan.blocks.size(),
                                    p->in, p->r, p->r_pad, reinterpret_cast<float *>(wsb + L.spart_off), Vbd,
                                    (__nv_bfloat16 *)V_save, st), 2);
        } else {
            CKL(launch_shrink_short((const __nv_bfloat16 *)X, p->d_slots, d_blocks, d_srows,
                                    (int)plan.blocks.size(), p->in, p->r, p->r_pad, Vbd, (__nv_bfloat16 *)V_save,
                                    st), 1);
        }
    }
    if (tiles.empty()) return SMLM_OK;
    const int bnw = kBN - p->r_pad;
    // long tiles on CTA pairs: consecutive tiles of one segment (same adapter) share one M=256 MMA
    int first_1cta = 0;  // tiles[first_1cta ..] go to the 1-CTA kernel
    if (has_w && p->cta_pair && !pairs.empty()) {
        Gemm2Args g2;
        memset(&g2, 0, sizeof(g2));
        if ((rc = make_map(&g2.tmX, X, p->in, b->S, 64, 128, CU_TENSOR_MAP_SWIZZLE_128B))) return rc;
        if ((rc = make_map(&g2.tmW0, W, p->in, p->out, 64, 128, CU_TENSOR_MAP_SWIZZLE_128B))) return rc;
        if ((rc = make_map(&g2.tmW1, W, p->in, p->out, 64, bnw - 128, CU_TENSOR_MAP_SWIZZLE_128B))) return rc;
        if (!plan.blocks.empty()) {
            if ((rc = make_map(&g2.tmU, Vbd, p->r_pad, plan.blocks.size() * 128, p->r_pad, 128,
                               swizzle_for(p->r_pad * 2))))
                return rc;
            g2.has_u = 1;
        }
        g2.blocks = d_blocks;
        g2.defer = getenv("SMLM_NO_DEFER") ? 0 : 1;
        g2.slots = p->d_slots;
        g2.pairs = reinterpret_cast<const DevPair *>(wsb + L.plan_off + pair_off);
        g2.n_pairs = (int)pairs.size();
        g2.n_ntiles = (p->out + bnw - 1) / bnw;
        g2.group_m = (raster_group(p->in) + 1) / 2;
        g2.K = p->in;
        g2.N = p->out;
        g2.r = p->r;
        g2.r_pad = p->r_pad;
        g2.stages = gemm2_stages(p->r_pad);
        g2.Y = Y;
        g2.Vsave = V_save;
        ProfScope ps(0, st);
        CKL(launch_gemm2(g2, false, p->num_sms, st), 1);
        first_1cta = (int)tiles.size();
    }
    if ((int)tiles.size() == first_1cta) return SMLM_OK;
    GemmArgs a;
    memset(&a, 0, sizeof(a));
    if ((rc = make_map(&a.tmA, X, p->in, b->S, 64, 128, CU_TENSOR_MAP_SWIZZLE_128B))) return rc;
    if (has_w && (rc = make_map(&a.tmB, W, p->in, p->out, 64, bnw, CU_TENSOR_MAP_SWIZZLE_128B))) return rc;
    if (!plan.blocks.empty() &&
        (rc = make_map(&a.tmV, Vbd, p->r_pad, plan.blocks.size() * 128, p->r_pad, 128, swizzle_for(p->r_pad * 2))))
        return rc;
    a.slots = p->d_slots;
    a.tiles = d_tiles + first_1cta;
    a.blocks = d_blocks;
    a.n_tiles = (int)tiles.size() - first_1cta;
    a.K = p->in;
    a.N = p->out;
    a.n_ntiles = (p->out + bnw - 1) / bnw;
    a.r = p->r;
    a.r_pad = p->r_pad;
    a.stages = gemm_stages(p->r_pad, nullptr);
    a.group_m = raster_group(p->in);
    a.has_w = has_w ? 1 : 0;
    a.Y = Y;
    a.Vsave = V_save;
    a.sUt = nullptr;
    a.S = b->S;
    {
        ProfScope ps(0, st);
        CKL(launch_gemm(a, false, p->num_sms, st), 1);
    }
    return SMLM_OK;
}

int smlm_backward(smlm_pool p, const smlm_batch *b, const void *X, const void *W, const void *dY, const void *V_save,
                  void *dX, int accumulate, void *ws, size_t ws_bytes, void *stream) {
    if (!p || !b) return set_err(SMLM_E_INVALID, "NULL pool/batch");
    Plan plan;
    int rc = plan_for(p, b, true, plan);
    if (rc) return rc;
    if (b->S == 0 || b->G == 0 || plan.bwd_tiles.empty()) return SMLM_OK;
    if (!X || !dY) return set_err(SMLM_E_INVALID, "X and dY must be non-NULL");
    if (dX && !W) return set_err(SMLM_E_INVALID, "W is required when dX is requested");
    WsLayout L = layout_for(p, b, plan, true, p->dtype == SMLM_FP32 || V_save == nullptr);
    if (!ws || ws_bytes < L.total) return set_err(SMLM_E_WORKSPACE, "workspace too small");
    DeviceGuard dg(p->device);
    if ((rc = check_sticky())) return rc;
    cudaStream_t st = (cudaStream_t)stream;
    uint8_t *wsb = reinterpret_cast<uint8_t *>(ws);

    // grad groups with the current grad bindings (masking: NULL => no dA/dB for that slot)
    std::vector<uint8_t> gbytes(plan.groups.size() * grad_group_bytes());
    int n_grad = 0;
    for (auto &g : plan.groups) {
        const SlotHost &h = p->slots[g.slot];
        if (!h.dA && !h.dB) continue;
        fill_grad_group(gbytes.data() + n_grad * grad_group_bytes(), g.slot, g.tile_begin, g.n_tiles, h.dA, h.dB);
        ++n_grad;
    }
    gbytes.resize(n_grad * grad_group_bytes());
    std::vector<int> uitems;
    for (size_t i = 0; i < plan.bwd_tiles.size(); ++i)
        if (plan.bwd_tiles[i].slot >= 0) uitems.push_back((int)i);
    // CTA pairs of consecutive fine-tune tiles of one segment (the dX GEMM on cta_group::2)
    std::vector<DevPair> bpairs;
    for (size_t i = 0; i < plan.bwd_tiles.size();) {
        const DevTile &t0 = plan.bwd_tiles[i];
        DevPair pr{};
        pr.row0 = t0.row0;
        pr.slot = t0.slot;
        pr.flags = kPairFT;
        pr.scale = t0.scale;
        pr.tile = (int)i;
        if (i + 1 < plan.bwd_tiles.size() && plan.bwd_tiles[i + 1].seg == t0.seg) {
            pr.rows = 128 + plan.bwd_tiles[i + 1].rows;
            i += 2;
        } else {
            pr.rows = t0.rows;
            i += 1;
        }
        bpairs.push_back(pr);
    }
    std::vector<uint8_t> bytes;
    append(bytes, plan.bwd_tiles);
    const size_t grp_off = bytes.size();
    bytes.insert(bytes.end(), gbytes.begin(), gbytes.end());
    const size_t uit_off = bytes.size();
    append(bytes, uitems);
    while (bytes.size() % 16) bytes.push_back(0);
    const size_t bpair_off = bytes.size();
    append(bytes, bpairs);
    if ((rc = stage_upload(p, bytes, wsb + L.plan_off, st))) return rc;
    const DevTile *d_tiles = reinterpret_cast<const DevTile *>(wsb + L.plan_off);
    const void *d_groups = wsb + L.plan_off + grp_off;
    const int *d_uitems = reinterpret_cast<const int *>(wsb + L.plan_off + uit_off);
    const DevPair *d_pairs = reinterpret_cast<const DevPair *>(wsb + L.plan_off + bpair_off);
    const int n_pairs = (int)bpairs.size();
    const int nt = (int)plan.bwd_tiles.size();
    float *Uf = reinterpret_cast<float *>(wsb + L.u_off);
    float *Vf = reinterpret_cast<float *>(wsb + L.vf_off);

    if (p->dtype == SMLM_FP32) {
        CKL(launch_rows_u<float>(d_tiles, nt, p->d_slots, (const float *)dY, p->out, p->r, Uf, nullptr, p->r_pad,
                                 st), 1);
        if (dX)
            CKL(launch_f32_dx(d_tiles, nt, p->d_slots, (const float *)dY, (const float *)W, (float *)dX, Uf, p->in,
                              p->out, p->r, st), 1);
        if (n_grad) {
            const float *V = (const float *)V_save;
            if (!V) {
                CKL(launch_rows_shrink<float>(d_tiles, nt, p->d_slots, (const float *)X, p->in, p->r, Vf, nullptr,
                                              0, st), 1);
                V = Vf;
            }
            CKL((launch_dadb<float, float>(d_tiles, d_groups, n_grad, (const float *)X, (const float *)dY, Uf, V,
                                           p->in, p->out, p->r, accumulate, st)), 2);
        }
        return SMLM_OK;
    }

    // ---------------- bf16 path ----------------
    __nv_bfloat16 *sUt = reinterpret_cast<__nv_bfloat16 *>(wsb + L.sut_off);
    __nv_bfloat16 *sVt = reinterpret_cast<__nv_bfloat16 *>(wsb + L.svt_off);
    // U = dY B_a per fine-tune tile (split-K tensor-core pass) -> tile-compact s*U
    if (L.u_items && (dX || n_grad)) {
        UArgs u;
        memset(&u, 0, sizeof(u));
        if ((rc = make_map(&u.tmDY, dY, p->out, b->S, 64, 128, CU_TENSOR_MAP_SWIZZLE_128B))) return rc;
        u.slots = p->d_slots;
        u.tiles = d_tiles;
        u.items = d_uitems;
        u.n_items = L.u_items;
        u.ksplit = L.u_ksplit;
        u.K = p->out;
        u.r_pad = p->r_pad;
        u.part = reinterpret_cast<float *>(wsb + L.upart_off);
        u.sUt = sUt;
        CKL(launch_u(u, p->num_sms, st), 2);
    }
    if (dX) {
        ProfScope ps(1, st);
        if (p->cta_pair) {
            Gemm2Args g2;
            memset(&g2, 0, sizeof(g2));
            if ((rc = make_map(&g2.tmX, dY, p->out, b->S, 64, 128, CU_TENSOR_MAP_SWIZZLE_128B))) return rc;
            if ((rc = make_map(&g2.tmW0, W, p->in, p->out, 64, 64, CU_TENSOR_MAP_SWIZZLE_128B))) return rc;
            if (L.u_items &&
                (rc = make_map(&g2.tmU, sUt, p->r_pad, (uint64_t)nt * 128, p->r_pad, 128, swizzle_for(p->r_pad * 2))))
                return rc;
            g2.has_u = L.u_items > 0;
            g2.slots = p->d_slots;
            g2.pairs = d_pairs;
            g2.n_pairs = n_pairs;
            g2.n_ntiles = (p->in + kBN - 1) / kBN;
            g2.group_m = (raster_group(p->out) + 1) / 2;
            g2.K = p->out;
            g2.N = p->in;
            g2.r = p->r;
            g2.r_pad = p->r_pad;
            g2.stages = gemm2_stages(p->r_pad);
            g2.Y = dX;
            g2.Vsave = nullptr;
            CKL(launch_gemm2(g2, true, p->num_sms, st), 1);
        } else {
            GemmArgs a;
            memset(&a, 0, sizeof(a));
            if ((rc = make_map(&a.tmA, dY, p->out, b->S, 64, 128, CU_TENSOR_MAP_SWIZZLE_128B))) return rc;
            if ((rc = make_map(&a.tmB, W, p->in, p->out, 64, 64, CU_TENSOR_MAP_SWIZZLE_128B))) return rc;
            if (L.u_items &&
                (rc = make_map(&a.tmV, sUt, p->r_pad, (uint64_t)nt * 128, p->r_pad, 128, swizzle_for(p->r_pad * 2))))
                return rc;
            a.slots = p->d_slots;
            a.tiles = d_tiles;
            a.blocks = nullptr;
            a.n_tiles = nt;
            a.K = p->out;
            a.N = p->in;
            a.n_ntiles = (p->in + kBN - 1) / kBN;
            a.r = p->r;
            a.r_pad = p->r_pad;
            a.stages = gemm_stages(p->r_pad, nullptr);
            a.group_m = raster_group(p->out);
            a.has_w = 1;
            a.Y = dX;
            a.Vsave = nullptr;
            a.sUt = nullptr;
            a.S = b->S;
            CKL(launch_gemm(a, true, p->num_sms, st), 1);
        }
    }
    if (n_grad) {
        ProfScope ps(3, st);
        if (V_save) {
            CKL(launch_prep_sv<__nv_bfloat16>(d_tiles, nt, (const __nv_bfloat16 *)V_save, p->r, p->r_pad, sVt, st), 1);
        } else {
            CKL(launch_rows_shrink<__nv_bfloat16>(d_tiles, nt, p->d_slots, (const __nv_bfloat16 *)X, p->in, p->r, Vf,
                                                  nullptr, 0, st), 1);
            CKL(launch_prep_sv<float>(d_tiles, nt, Vf, p->r, p->r_pad, sVt, st), 1);
        }
        TokArgs ta;
        memset(&ta, 0, sizeof(ta));
        const int rb = p->r_pad * 2;
        if ((rc = make_map(&ta.tmX, X, p->in, b->S, 64, 64, CU_TENSOR_MAP_SWIZZLE_128B))) return rc;
        if ((rc = make_map(&ta.tmDY, dY, p->out, b->S, 64, 64, CU_TENSOR_MAP_SWIZZLE_128B))) return rc;
        if ((rc = make_map(&ta.tmSU, sUt, p->r_pad, (uint64_t)nt * 128, p->r_pad, 64, swizzle_for(rb)))) return rc;
        if ((rc = make_map(&ta.tmSV, sVt, p->r_pad, (uint64_t)nt * 128, p->r_pad, 64, swizzle_for(rb)))) return rc;
        ta.tiles = d_tiles;
        ta.groups = reinterpret_cast<const GradGroup *>(d_groups);
        ta.n_groups = n_grad;
        ta.in_f = p->in;
        ta.out_f = p->out;
        ta.r = p->r;
        ta.r_pad = p->r_pad;
        ta.mt_a = (p->in + 127) / 128;
        ta.mt_b = (p->out + 127) / 128;
        ta.accumulate = accumulate ? 1 : 0;
        CKL(launch_tok(ta, p->num_sms, st), 1);
    }
    return SMLM_OK;
}

}  // extern "C"
