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

#include <stdio.h>

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
                        __nv_bfloat16 *Vsave, const DropArgs &drop, cudaStream_t st);
template <typename T>
int launch_rows_shrink(const DevTile *tiles, int n_tiles, const SlotDev *slots, const T *X, int in_f, int r,
                       float *Vf, T *Vsave, int ft_only, const DropArgs &drop, cudaStream_t st);
template <typename T>
int launch_rows_u(const DevTile *tiles, int n_tiles, const SlotDev *slots, const T *dY, int out_f, int r, float *Uf,
                  __nv_bfloat16 *sUt, int r_pad, cudaStream_t st);
template <typename TV>
int launch_prep_sv(const DevTile *tiles, int n_tiles, const TV *V, int r, int r_pad, __nv_bfloat16 *sVt,
                   cudaStream_t st);
int launch_tok(const TokArgs &a, int num_sms, cudaStream_t st);
int dec_chunks(int in_f);
int dec3_stages();
int dec3_max_clusters(int r_pad);
int launch_dec3(const Dec3Args &a, const Dec3Inline &in, int clusters, cudaStream_t st);
int launch_plan_copy(void *dst, const void *src, size_t n, cudaStream_t st);
int adamw_grid(int num_sms, size_t n);
int launch_adamw_sumsq(const AdamwArgs &a, float *partial, int grid, cudaStream_t st);
int launch_fanout_signal(const FanoutFlags &f, cudaStream_t st);
int launch_fanout_wait(const int *ready, int target, cudaStream_t st);
int launch_attn(const AttnArgs &a, const AttnDecInline &dinl, int n_items, int n_rows, int n_drows, int n_dgroups,
                cudaStream_t st);
int launch_adamw_step(const AdamwArgs &a, int grid, cudaStream_t st);
int launch_shrink_split(const __nv_bfloat16 *X, const SlotDev *slots, const DevBlock *blocks,
                        const DevShortRow *srows, int n_blocks, int in_f, int r, int r_pad, float *part,
                        __nv_bfloat16 *Vbd, __nv_bfloat16 *Vsave, int *ctr, const DropArgs &drop, cudaStream_t st);
size_t grad_group_bytes();
void fill_grad_group(void *dst, int slot, int tile_begin, int n_tiles, int r, float *dA, float *dB);
template <typename T, typename TV>
int launch_dadb(const DevTile *tiles, const void *groups, int n_groups, const T *X, const T *dY, const float *Uf,
                const TV *V, int in_f, int out_f, int r, int accumulate, const DropArgs &drop, cudaStream_t st);
int launch_f32_fwd(const DevTile *tiles, int n_tiles, const SlotDev *slots, const float *X, const float *W, float *Y,
                   const float *Vf, int in_f, int out_f, int r, cudaStream_t st);
int launch_f32_dx(const DevTile *tiles, int n_tiles, const SlotDev *slots, const float *dY, const float *W, float *dX,
                  const float *Uf, int in_f, int out_f, int r, const DropArgs &drop, cudaStream_t st);
}  // namespace smlm

using namespace smlm;

// ------------------------------------------------------------------------------------------
// error reporting, instrumentation
// ------------------------------------------------------------------------------------------
static thread_local std::string g_last_error;
static std::atomic<uint64_t> g_launches{0};

// Measurement-only switches exist only in a library built with -DSMLM_MEASURE (build.py --measure
// -> libsmlm_measure.so); the release library reads no environment variable.  None of them
// changes a result: SMLM_HOST_PROF prints host phase times, SMLM_DEC3_DEBUG records per-CTA
// phase timestamps of the decode kernel in the workspace tail.
#include <chrono>
#include <cmath>
#ifdef SMLM_MEASURE
static bool measure_flag(const char *name) {
    const char *e = getenv(name);
    return e && *e && strcmp(e, "0") != 0;
}
static int measure_int(const char *name, int dflt) {
    const char *e = getenv(name);
    return e && *e ? atoi(e) : dflt;
}
#else
static constexpr bool measure_flag(const char *) { return false; }
static constexpr int measure_int(const char *, int dflt) { return dflt; }
#endif
struct HostProf {
    bool on = measure_flag("SMLM_HOST_PROF");
    double t[8] = {0};
    long n = 0;
    ~HostProf() {
        if (on && n)
            fprintf(stderr, "[smlm host] calls=%ld plan=%.2f dec3plan=%.2f upload=%.2f maps=%.2f launch=%.2f us/call\n", n,
                    t[0] / n, t[1] / n, t[2] / n, t[3] / n, t[4] / n);
    }
} g_hprof;
static inline double now_us() {
    return std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

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
    int r = 0;   // the adapter's rank (<= pool rank)
};

size_t align256(size_t x) { return (x + 255) & ~size_t(255); }

// m-tiles per raster group: the group's 128-row A tiles (128 x K bf16) stay L2-resident while
// the CTAs sweep every n-tile, so each W n-tile is fetched from HBM once per group (~48 MB budget)
int raster_group(int K) {
    const long tile = 128L * K * 2;
    long g = ((long)measure_int("SMLM_RASTER_BWD_MB", 48) << 20) / tile;
    if (g < 4) g = 4;
    if (g > 64) g = 64;
    return (int)g;
}
// CTA-pair GEMMs: pairs per raster group -- a ~24 MB budget of X tiles, then the groups
// balanced (53 pairs at K = 4096: 5 groups of 11 / 10).  The L2 is two ~63 MB halves, one per
// die, and the X band of a group is read from both: a 64 MB band (2 W passes on paper) measured
// 3.2 GB of DRAM traffic for the C4 gate/up launch and 2.13 M tokens/s, 24 MB 2.4 GB and
// 2.18-2.19 M (same box, scripts/sweep_raster.sh)
int raster_group_pairs(int K, int n_pairs) {
    const long pair = 256L * K * 2;
    long g = ((long)measure_int("SMLM_RASTER_MB", 24) << 20) / pair;
    if (g < 2) g = 2;
    if (g > 64) g = 64;
    const long groups = (n_pairs + g - 1) / g;
    return (int)std::max<long>(1, (n_pairs + groups - 1) / groups);
}

}  // namespace

struct smlm_pool_s {
    int device = 0;
    int in = 0, out = 0, r = 0, r_pad = 16, cap = 0, dtype = 0;
    int l_long = 64;
    int cta_pair = 1;   // forward long tiles on CTA pairs (cta_group::2)
    int dec_kernel = 1; // pure decode batches take the single-launch decode kernel (SMLM_OPT_DECODE_KERNEL)
    int dec_ksplit = 0; // decode W split-K factor, 0 = automatic (SMLM_OPT_DEC_KSPLIT)
    int dec_coop = 0;   // cooperative decode launches (SMLM_OPT_DEC_COOPERATIVE)
    std::vector<long long> fanout;   // dA/dB also stored at p + delta (peer ranks' staging slots, f3)
    int num_sms = 148;
    std::vector<SlotHost> slots;
    std::vector<uint8_t> ok;
    std::vector<float> scales;
    SlotDev *d_slots = nullptr;
    // self-resetting cross-CTA counters, one set per launching stream (calls on one stream are
    // ordered; calls of one pool on different streams -- e.g. the next micro-batch's forward
    // overlapping this one's backward -- must not share them): [0, dec3_counter_ints()) decode
    // kernel, then kUCtrMax per-item split counters of the U / pre-shrink / short-shrink passes
    struct CtrSet { cudaStream_t st; int *d; };
    std::vector<CtrSet> ctrs;
    // encoded TMA descriptors of recently used (pointer, shape, box) keys: steady-state calls reuse them
    struct MapEnt {
        const void *ptr;
        uint64_t inner, outer;
        uint32_t b0, b1;
        int swz;
        CUtensorMap map;
    };
    std::vector<MapEnt> map_cache;
    size_t map_next = 0;
    Ring ring;
    // pinned arena for plan uploads recorded into a CUDA graph (stream capture): a captured memcpy
    // node re-reads its host source at every replay, so captured plans get their own bytes that live
    // until the pool is destroyed (bump allocation; no event synchronisation during capture)
    uint8_t *cap_arena = nullptr;
    size_t cap_used = 0, cap_size = 0;
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

// The pool's counter set of stream `st`: pool_create pre-allocates kCtrSets zeroed sets that are
// bound to streams on first use (no allocation or memset on the call path, so calls can be
// captured into CUDA graphs); more streams allocate further sets outside graph capture.
constexpr int kCtrSets = 4;
size_t ctr_set_ints() { return (size_t)dec3_counter_ints() + kUCtrMax; }
int stream_counters(smlm_pool p, cudaStream_t st, int **dec_ctr, int **u_ctr) {
    int *d = nullptr;
    for (auto &c : p->ctrs)
        if (c.d && c.st == st) d = c.d;
    if (!d)
        for (auto &c : p->ctrs)
            if (c.d && c.st == (cudaStream_t)-1) {   // a free pre-allocated set
                c.st = st;
                d = c.d;
                break;
            }
    if (!d) {
        cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
        cudaStreamIsCapturing(st, &cs);
        if (cs != cudaStreamCaptureStatusNone)
            return set_err(SMLM_E_UNSUPPORTED, "graph capture on a new stream: this pool already serves its maximum of "
                                               "streams; issue one call on the stream outside capture first");
        cudaError_t e = cudaMalloc(&d, ctr_set_ints() * sizeof(int));
        if (e != cudaSuccess) return cuda_err(e, "cudaMalloc(counters)");
        e = cudaMemset(d, 0, ctr_set_ints() * sizeof(int));
        if (e != cudaSuccess) {
            cudaFree(d);
            return cuda_err(e, "cudaMemset(counters)");
        }
        p->ctrs.push_back({st, d});
    }
    if (dec_ctr) *dec_ctr = d;
    if (u_ctr) *u_ctr = d + dec3_counter_ints();
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
    size_t pre_sv_off = 0, pre_sv_bytes = 0;     // bf16 fwd: pre-shrunk s*V of the long tiles
    size_t pre_part_off = 0, pre_part_bytes = 0; // bf16 fwd: its split-K partials
    int pre_items = 0, pre_ksplit = 0;
    size_t total = 0;
};

// split-K factor of the U / pre-shrink pass: about one work unit per SM, >= 4 K-blocks per unit
// (measured against ~4 units per SM with >= 8 K-blocks: finer splits cost more partial traffic
// and power than they gain in balance, 1-2 % of the C4 step)
static int u_ksplit(int num_sms, int items, int nkb) {
    int ks = num_sms / items;
    if (ks > nkb / 4) ks = nkb / 4;
    return ks < 1 ? 1 : ks;
}

// set by smlm_forward_multi around its per-projection smlm_forward calls: s*V of the long tiles
// was already computed for every projection in one shared pass (f1 for mixed batches)
static thread_local const void *t_ext_pre_sv = nullptr;

// forward pre-shrink (s*V once per long tile, then full 256-column W tiles; DESIGN K1) on the
// CTA-pair path (the 1-CTA kernel keeps the shrink fused into its N=256 MMA)
static bool use_preshrink(smlm_pool p) { return p->dtype == SMLM_BF16 && p->cta_pair; }

int plan_for(smlm_pool p, const smlm_batch *b, bool bwd, Plan &plan) {
    std::string msg;
    // fp32 test mode consumes segment-aligned tiles for every row (L_long = 1)
    int l_long = p->dtype == SMLM_FP32 ? 1 : p->l_long;
    int rc = build_plan(b, p->cap, p->ok.data(), p->scales.data(), l_long, bwd, plan, msg);
    if (rc != SMLM_OK) return set_err(rc, msg);
    return SMLM_OK;
}

// LoRA dropout of the batch's FINETUNE rows (smlm.h smlm_batch; R13)
DropArgs make_drop(const smlm_batch *b, int in_f) {
    DropArgs d;
    memset(&d, 0, sizeof(d));
    const double pq = std::floor((double)b->dropout_p * 65536.0 + 0.5);   // round(p * 65536), p in [0, 1)
    d.thr = (uint32_t)std::min(pq, 65535.0);
    d.on = d.thr > 0;
    d.s0 = (uint32_t)(b->dropout_seed & 0xffffffffu);
    d.s1 = (uint32_t)(b->dropout_seed >> 32);
    d.half_in = (uint32_t)((in_f + 1) / 2);
    d.scale = (float)(65536.0 / (65536.0 - (double)d.thr));
    return d;
}
// does the plan have fine-tune rows with an adapter (the rows dropout acts on)?
bool has_ft_lora(const Plan &plan) {
    for (auto &t : plan.long_tiles)
        if (t.flags & kTileFT) return true;
    for (auto &r : plan.short_rows)
        if (r.ft) return true;
    for (auto &t : plan.bwd_tiles)
        if (t.slot >= 0) return true;
    return false;
}
// projection i of a multi-projection call draws an independent mask (PEFT: one dropout per module)
smlm_batch batch_for_projection(const smlm_batch *b, int i) {
    smlm_batch c = *b;
    c.dropout_seed = b->dropout_seed + (uint64_t)i * 0x9E3779B97F4A7C15ull;
    return c;
}

// make_map through the pool's small descriptor cache (round-robin replacement, 64 entries)
int make_map_cached(smlm_pool p, CUtensorMap *m, const void *ptr, uint64_t inner, uint64_t outer, uint32_t b0,
                    uint32_t b1, CUtensorMapSwizzle swz) {
    for (auto &e : p->map_cache)
        if (e.ptr == ptr && e.inner == inner && e.outer == outer && e.b0 == b0 && e.b1 == b1 && e.swz == (int)swz) {
            *m = e.map;
            return SMLM_OK;
        }
    int rc = make_map(m, ptr, inner, outer, b0, b1, swz);
    if (rc) return rc;
    smlm_pool_s::MapEnt e{ptr, inner, outer, b0, b1, (int)swz, *m};
    if (p->map_cache.size() < 64) {
        p->map_cache.push_back(e);
    } else {
        p->map_cache[p->map_next] = e;
        p->map_next = (p->map_next + 1) % 64;
    }
    return SMLM_OK;
}

// ------------------------------------------------------------------------------------------
// decode path v3 (kernels_dec3.cu): pure short batches of <= 512 rows, one or several
// projections that share X in one launch.
// ------------------------------------------------------------------------------------------
struct Dec3Plan {
    bool ok = false;
    std::vector<int> uslot;
    std::vector<Dec3RowInfo> rows;
    int n_groups = 0, nw = 0, n_vt = 0, ks = 1, ks_v = 1, n_vpairs = 0, n_wpairs = 0, clusters = 0;
    size_t plan_off = 0, sv_off[kDec3MaxProj] = {}, kpart_off = 0, total = 0;
};

// pools[0..n) share in, r and dtype (validated by the caller); every batch slot is registered in
// all of them.  ok = false if the batch cannot take the single-launch kernel.
Dec3Plan dec3_plan(int n_proj, const smlm_pool *pools, const smlm_batch *b, const Plan &plan) {
    Dec3Plan D;
    smlm_pool p0 = pools[0];
    if (p0->dtype != SMLM_BF16 || !plan.long_tiles.empty() || plan.short_tiles.empty() || b->S > kDec3InlineRows ||
        !p0->dec_kernel || (b->dropout_p > 0.f && has_ft_lora(plan)))   // dropout rows: the mixed path
        return D;
    // adapters of the batch (ascending) and per-row records
    D.rows.assign(b->S, Dec3RowInfo{-1, 0.f, 0, 0});
    std::vector<int> row_slot(b->S, -1);
    std::vector<uint8_t> present(p0->cap, 0);
    for (auto &bk : plan.blocks) {
        present[bk.slot] = 1;
        for (int i = 0; i < bk.nrows; ++i) {
            const DevShortRow &sr = plan.short_rows[bk.row_begin + i];
            row_slot[sr.row] = bk.slot;
            D.rows[sr.row].scale = sr.scale;
            D.rows[sr.row].ft = sr.ft;
        }
    }
    std::vector<int> uidx(p0->cap, -1);
    for (int sl = 0; sl < p0->cap; ++sl)
        if (present[sl]) {
            uidx[sl] = (int)D.uslot.size();
            D.uslot.push_back(sl);
        }
    for (int r = 0; r < b->S; ++r)
        if (row_slot[r] >= 0) D.rows[r].uidx = uidx[row_slot[r]];
    const int n_uniq = (int)D.uslot.size();
    if (n_uniq > kDec3InlineSlots) return D;
    D.n_groups = (b->S + 255) / 256;
    for (int i = 0; i < n_proj; ++i) D.nw += (pools[i]->out + 255) / 256;
    D.n_vt = (n_uniq * p0->r_pad + 255) / 256;
    // one co-resident wave (the kernel spin-waits across CTAs; launched cooperatively)
    const int pairs = std::min(std::min(p0->num_sms / 2, kDec3MaxPairs), dec3_max_clusters(p0->r_pad));
    if (pairs < 2) return D;
    const int NW = D.n_groups * D.nw, NV = D.n_groups * n_proj * D.n_vt;
    const int nkb = p0->in / kBK;
    const int kmax = std::max(1, std::min(8, nkb / 2));
    // split factors.  The W split depends only on the W tiles (so that B = 0 reproduces the
    // base-only call bit for bit: same K ranges, same summation order), taking ~3/4 of the wave;
    // the V tiles (shrink) get the rest, as many splits as fit (they must publish before the W
    // tiles finish their main loop)
    int best_ks = std::max(1, std::min(kmax, (pairs * 3 / 4) / std::max(NW, 1)));
    if (p0->dec_ksplit > 0)   // pool option SMLM_OPT_DEC_KSPLIT (tests: every split count is parity-checked)
        best_ks = std::max(1, std::min(p0->dec_ksplit, kmax));
    while (best_ks > 1 && NW * best_ks + NV > pairs) --best_ks;   // (only with very many adapters)
    // V splits (up to 16): fewer K-blocks per split keep all of a split's loads in
    // flight in the 6-stage ring (the V chain is load-latency bound, not bandwidth bound)
    const int kmax_v = std::max(1, std::min(16, nkb / 2));
    int best_ksv = NV ? std::max(1, std::min(kmax_v, (pairs - NW * best_ks) / NV)) : 1;
    if (NW * best_ks + NV * best_ksv > pairs) best_ks = 0;
    if (best_ks == 0) return D;   // more tiles than one wave: not this kernel
    D.ks = best_ks;
    D.ks_v = NV ? best_ksv : 1;
    D.n_vpairs = NV * D.ks_v;
    D.n_wpairs = NW * D.ks;
    D.clusters = D.n_vpairs + D.n_wpairs;
    if (NV + NW > 256) return D;   // tile arrival counters
    size_t off = 0;
    D.plan_off = off;
    off = align256(off + (size_t)n_uniq * 4 + 64 + D.rows.size() * sizeof(Dec3RowInfo));
    for (int i = 0; i < n_proj; ++i) {
        D.sv_off[i] = off;
        off = align256(off + (size_t)D.n_groups * std::max(n_uniq, 1) * 256 * p0->r_pad * 2);
    }
    D.kpart_off = off;
    off = align256(off + (size_t)D.clusters * 2 * 8 * kDec3ChunkBytes);
    if (measure_flag("SMLM_DEC3_DEBUG")) off += 2 * kDec3MaxPairs * 16 * 8;   // phase timestamps at the tail
    D.total = off;
    D.ok = true;
    return D;
}

WsLayout layout_for(smlm_pool p, const smlm_batch *b, const Plan &plan, bool bwd, bool need_vf) {
    WsLayout L;
    size_t off = 0;
    if (!bwd) {
        L.plan_bytes = (plan.long_tiles.size() + plan.short_tiles.size()) * sizeof(DevTile) +
                       plan.blocks.size() * sizeof(DevBlock) + plan.short_rows.size() * sizeof(DevShortRow) + 16 +
                       (plan.long_tiles.size() + plan.short_tiles.size()) * sizeof(DevPair) + 16 +
                       plan.long_tiles.size() * sizeof(int) + 16;
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
        if (use_preshrink(p)) {
            for (auto &t : plan.long_tiles)
                if (t.slot >= 0) ++L.pre_items;
            if (L.pre_items) {
                const int ks = u_ksplit(p->num_sms, L.pre_items, p->in / 64);
                L.pre_ksplit = ks;
                L.pre_sv_off = off;
                L.pre_sv_bytes = plan.long_tiles.size() * 128 * (size_t)p->r_pad * 2;
                off = align256(off + L.pre_sv_bytes);
                L.pre_part_off = off;
                L.pre_part_bytes = (size_t)L.pre_items * ks * 128 * p->r_pad * 4;
                off = align256(off + L.pre_part_bytes);
            }
        }
    }
    if (!bwd) {
        const Dec3Plan D = dec3_plan(1, &p, b, plan);
        if (D.ok) off = std::max(off, D.total);   // the decode path uses its own layout from offset 0
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
            const int ks = u_ksplit(p->num_sms, L.u_items, p->out / 64);
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
// via_memcpy: always a copy-engine transfer (slot-table updates: TMA descriptors must never be
// written by a kernel that its PDL successors overlap)
int stage_upload(smlm_pool p, const std::vector<uint8_t> &bytes, void *dst, cudaStream_t st, bool via_memcpy = false) {
    if (bytes.empty()) return SMLM_OK;
    if (!via_memcpy) {
        // small plans ride in kernel parameters (kernels_plan.cu): never queued behind bulk DMA
        const int rc = launch_plan_copy(dst, bytes.data(), bytes.size(), st);
        if (rc == 0) {
            ++g_launches;
            return SMLM_OK;
        }
        if (rc > 0) return cuda_err((cudaError_t)rc, "plan upload (parameter copy)");
    }
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
    cudaStreamIsCapturing(st, &cs);
    if (cs != cudaStreamCaptureStatusNone) {
        const size_t need = (bytes.size() + 255) & ~size_t(255);
        if (!p->cap_arena || p->cap_used + need > p->cap_size)
            return set_err(SMLM_E_UNSUPPORTED, "graph capture: plan arena exhausted (call once outside capture to size it, "
                                               "or capture fewer calls per pool)");
        uint8_t *h = p->cap_arena + p->cap_used;
        p->cap_used += need;
        memcpy(h, bytes.data(), bytes.size());
        cudaError_t e = cudaMemcpyAsync(dst, h, bytes.size(), cudaMemcpyHostToDevice, st);
        if (e != cudaSuccess) return cuda_err(e, "plan upload (capture)");
        return SMLM_OK;
    }
    if (!p->cap_arena) {   // sized once, outside capture: room for many captured calls of this size
        p->cap_size = std::max<size_t>(1 << 20, 64 * ((bytes.size() + 255) & ~size_t(255)));
        if (cudaMallocHost((void **)&p->cap_arena, p->cap_size) != cudaSuccess) {
            p->cap_arena = nullptr;
            p->cap_size = 0;
        }
    }
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

int run_dec3(int n_proj, const smlm_pool *pools, const smlm_batch *b, const Dec3Plan &D, const void *X,
             const void *const *W, void *const *Y, void *const *Vsave, uint8_t *wsb, cudaStream_t st) {
    smlm_pool p0 = pools[0];
    const int n_uniq = (int)D.uslot.size();
    int rc;
    double t0 = g_hprof.on ? now_us() : 0;
    // the plan rides in the kernel parameters (sizes bounded by dec3_plan: <= 256 adapters, <= 512 rows)
    static thread_local Dec3Inline inl;
    if (n_uniq) memcpy(inl.uslot, D.uslot.data(), n_uniq * sizeof(int));
    if (!D.rows.empty()) memcpy(inl.rows, D.rows.data(), D.rows.size() * sizeof(Dec3RowInfo));
    double t1 = g_hprof.on ? now_us() : 0;
    int *ctr = nullptr;
    if ((rc = stream_counters(p0, st, &ctr, nullptr))) return rc;
    Dec3Args a;
    memset(&a, 0, sizeof(a));
    if ((rc = make_map_cached(p0, &a.tmX, X, p0->in, b->S, 64, 128, CU_TENSOR_MAP_SWIZZLE_128B))) return rc;
    int nt0 = 0;
    for (int i = 0; i < n_proj; ++i) {
        Dec3Proj &P = a.proj[i];
        if ((rc = make_map_cached(p0, &P.tmW, W[i], p0->in, pools[i]->out, 64, 128, CU_TENSOR_MAP_SWIZZLE_128B)))
            return rc;
        if ((rc = make_map_cached(p0, &P.tmY, Y[i], pools[i]->out, b->S, 32, 128, CU_TENSOR_MAP_SWIZZLE_NONE)))
            return rc;
        P.sv = wsb + D.sv_off[i];
        if (n_uniq > 0 && (rc = make_map_cached(p0, &P.tmSV, P.sv, p0->r_pad, (uint64_t)D.n_groups * n_uniq * 256,
                                                p0->r_pad, 128, swizzle_for(p0->r_pad * 2))))
            return rc;
        P.slots = pools[i]->d_slots;
        P.Vsave = Vsave ? Vsave[i] : nullptr;
        P.out = pools[i]->out;
        P.nt0 = nt0;
        P.n_wt = (pools[i]->out + 255) / 256;
        nt0 += P.n_wt;
    }
    a.kpart = reinterpret_cast<float *>(wsb + D.kpart_off);
    a.ctr = ctr;
    a.n_proj = n_proj;
    a.n_uniq = n_uniq;
    a.n_groups = D.n_groups;
    a.n_wt = D.nw;
    a.n_vt = D.n_vt;
    a.ks = D.ks;
    a.ks_v = D.ks_v;
    a.n_vpairs = D.n_vpairs;
    a.n_wpairs = D.n_wpairs;
    a.S = b->S;
    a.K = p0->in;
    a.r = p0->r;
    a.r_pad = p0->r_pad;
    a.stages = dec3_stages();
    a.cooperative = p0->dec_coop;
    if (measure_flag("SMLM_DEC3_DEBUG"))
        a.dbg = reinterpret_cast<unsigned long long *>(wsb + D.total - 2 * kDec3MaxPairs * 16 * 8);
    double t2 = g_hprof.on ? now_us() : 0;
    {
        ProfScope ps(0, st);
        CKL(launch_dec3(a, inl, D.clusters, st), 1);
    }
    if (g_hprof.on) {
        g_hprof.t[2] += t1 - t0;
        g_hprof.t[3] += t2 - t1;
        g_hprof.t[4] += now_us() - t2;
    }
    return SMLM_OK;
}

// ------------------------------------------------------------------------------------------
// bf16 forward: plan upload + short-row shrink (everything but the GEMM), and the CTA-pair GEMM
// arguments for one or several projections that share X and the batch
// ------------------------------------------------------------------------------------------
struct FwdPrep {
    int n_tiles = 0, n_long = 0, n_pairs = 0, n_pre_items = 0, n_blocks = 0;
    const DevTile *tiles_dev = nullptr;
    const DevBlock *blocks_dev = nullptr;
    const DevPair *pairs_dev = nullptr;   // set when the CTA-pair GEMM runs (W != NULL, cta_pair)
    const int *pre_items_dev = nullptr;
    __nv_bfloat16 *vbd = nullptr;          // block-diagonal s*V of the short tiles
    const SlotDev *slots = nullptr;
};

// A CTA pair takes two CONSECUTIVE tiles of the kept list (long tiles in segment order, then the
// short tiles), whatever their segments: only the partial 128-row tile at each segment end is
// padding (DESIGN K1).  An odd tile count leaves one half empty.
static DevHalf half_of(const DevTile &t, int idx) {
    DevHalf h{};
    h.row0 = t.row0;
    h.rows = t.rows;
    if (t.flags & kTileShort) {
        h.slot = -1;
        h.flags = kPairShort;
        h.blk0 = t.blk0;
        h.nblk = t.nblk;
    } else {
        h.slot = t.slot;
        h.flags = (t.flags & kTileFT) ? kPairFT : 0;
        h.scale = t.scale;
        h.tile = idx;
    }
    return h;
}
static void make_pairs(const std::vector<DevTile> &tiles, std::vector<DevPair> &pairs) {
    pairs.clear();
    for (size_t i = 0; i < tiles.size(); i += 2) {
        DevPair pr{};
        pr.h[0] = half_of(tiles[i], (int)i);
        if (i + 1 < tiles.size()) {
            pr.h[1] = half_of(tiles[i + 1], (int)i + 1);
        } else {
            pr.h[1] = pr.h[0];
            pr.h[1].rows = 0;
            pr.h[1].slot = -1;
            pr.h[1].flags = 0;
            pr.h[1].nblk = 0;
        }
        pairs.push_back(pr);
    }
}

static int fwd_prepare(smlm_pool p, const smlm_batch *b, const Plan &plan, const WsLayout &L, const void *X,
                       const void *W, void *V_save, uint8_t *wsb, int *uctr, cudaStream_t st, FwdPrep &F) {
    int rc;
    const bool has_w = W != nullptr;
    std::vector<DevTile> tiles;
    tiles.reserve(plan.long_tiles.size() + plan.short_tiles.size());
    for (auto &t : plan.long_tiles)
        if (has_w || (t.flags & kTileLora)) tiles.push_back(t);
    F.n_long = (int)tiles.size();
    for (auto &t : plan.short_tiles)
        if (has_w || t.nblk > 0) tiles.push_back(t);
    F.n_tiles = (int)tiles.size();
    std::vector<DevPair> pairs;
    const bool pair_gemm = has_w && p->cta_pair;
    if (pair_gemm) make_pairs(tiles, pairs);
    std::vector<int> pre_items;   // long tiles with an adapter (pre-shrink work items)
    if (pair_gemm && use_preshrink(p))
        for (int i = 0; i < F.n_long; ++i)
            if (tiles[i].slot >= 0) pre_items.push_back(i);
    std::vector<uint8_t> bytes;
    append(bytes, tiles);
    const size_t blk_off = bytes.size();
    append(bytes, plan.blocks);
    const size_t srow_off = bytes.size();
    append(bytes, plan.short_rows);
    while (bytes.size() % 16) bytes.push_back(0);
    const size_t pair_off = bytes.size();
    append(bytes, pairs);
    const size_t pre_off = bytes.size();
    append(bytes, pre_items);
    F.tiles_dev = reinterpret_cast<const DevTile *>(wsb + L.plan_off);
    F.blocks_dev = reinterpret_cast<const DevBlock *>(wsb + L.plan_off + blk_off);
    const DevShortRow *d_srows = reinterpret_cast<const DevShortRow *>(wsb + L.plan_off + srow_off);
    F.pairs_dev = pair_gemm ? reinterpret_cast<const DevPair *>(wsb + L.plan_off + pair_off) : nullptr;
    F.pre_items_dev = reinterpret_cast<const int *>(wsb + L.plan_off + pre_off);
    F.n_pairs = (int)pairs.size();
    F.n_pre_items = (int)pre_items.size();
    F.n_blocks = (int)plan.blocks.size();
    F.vbd = reinterpret_cast<__nv_bfloat16 *>(wsb + L.vbd_off);
    F.slots = p->d_slots;
    if ((rc = stage_upload(p, bytes, wsb + L.plan_off, st))) return rc;
    if (!plan.blocks.empty()) {
        ProfScope ps(2, st);
        if (L.spart_bytes) {
            // the last chunk of each block combines it in-kernel (stream counters, self-resetting)
            int *sctr = (int)plan.blocks.size() <= kUCtrMax ? uctr : nullptr;
            CKL(launch_shrink_split((const __nv_bfloat16 *)X, p->d_slots, F.blocks_dev, d_srows,
                                    (int)plan.blocks.size(), p->in, p->r, p->r_pad,
                                    reinterpret_cast<float *>(wsb + L.spart_off), F.vbd, (__nv_bfloat16 *)V_save,
                                    sctr, make_drop(b, p->in), st), sctr ? 1 : 2);
        } else {
            CKL(launch_shrink_short((const __nv_bfloat16 *)X, p->d_slots, F.blocks_dev, d_srows,
                                    (int)plan.blocks.size(), p->in, p->r, p->r_pad, F.vbd, (__nv_bfloat16 *)V_save,
                                    make_drop(b, p->in), st), 1);
        }
    }
    return SMLM_OK;
}

// CTA-pair GEMM arguments for n_proj projections (pools share in / r / dtype and the batch plan):
// F[i] from fwd_prepare of projection i (its own workspace: short-tile s*V), pre_sv[i] its
// tile-compact s*V of the long tiles.  The pairs / tiles of F[0] serve every projection.
static int gemm2_fwd_args(int n_proj, const smlm_pool *pools, const smlm_batch *b, const void *X,
                          const void *const *W, void *const *Y, const FwdPrep *F, __nv_bfloat16 *const *pre_sv,
                          Gemm2Args &g2) {
    int rc;
    smlm_pool p0 = pools[0];
    memset(&g2, 0, sizeof(g2));
    int nt0 = 0;
    for (int i = 0; i < n_proj; ++i) {
        smlm_pool pi = pools[i];
        Gemm2Proj &P = g2.proj[i];
        if ((rc = make_map_cached(p0, &P.tmA, X, p0->in, b->S, 64, 128, CU_TENSOR_MAP_SWIZZLE_128B))) return rc;
        P.K = p0->in;
        if ((rc = make_map_cached(p0, &P.tmW, W[i], pi->in, pi->out, 64, 128, CU_TENSOR_MAP_SWIZZLE_128B))) return rc;
        const uint32_t rp = (uint32_t)pi->r_pad;
        if (F[i].n_blocks) {
            if ((rc = make_map(&P.tmU, F[i].vbd, rp, (uint64_t)F[i].n_blocks * 128, rp, 128, swizzle_for(rp * 2))))
                return rc;
            P.has_u = 1;
            P.u_rows = F[i].n_blocks * 128;
        }
        if (F[i].n_pre_items) {
            if ((rc = make_map(&P.tmV, pre_sv[i], rp, (uint64_t)F[i].n_long * 128, rp, 128, swizzle_for(rp * 2))))
                return rc;
            P.has_v = 1;
            P.v_rows = F[i].n_long * 128;
        }
        P.slots = pi->d_slots;
        P.Y = Y[i];
        if ((rc = make_map_cached(p0, &P.tmY, Y[i], pi->out, b->S, 64, 128, CU_TENSOR_MAP_SWIZZLE_128B))) return rc;
        P.N = pi->out;
        P.nt0 = nt0;
        nt0 += (pi->out + kBN - 1) / kBN;
    }
    g2.pairs = F[0].pairs_dev;
    g2.blocks = F[0].blocks_dev;
    g2.n_proj = n_proj;
    g2.n_pairs = F[0].n_pairs;
    g2.n_nt = nt0;
    g2.group_m = raster_group_pairs(p0->in, F[0].n_pairs);
    g2.dbg = measure_flag("SMLM_GEMM2_DEBUG");
    g2.r = p0->r;
    g2.r_pad = p0->r_pad;
    g2.stages = gemm2_stages(p0->r_pad);
    return SMLM_OK;
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

// ---- AdamW step over the fine-tune adapters' flat parameters ----
static int current_sm100_sms(int *num_sms) {
    static thread_local int cached_dev = -1, cached_sms = 0;
    int dev = -1;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return set_err(SMLM_E_UNSUPPORTED, "no CUDA device (there is no CPU fallback)");
    if (dev != cached_dev) {
        cudaDeviceProp prop;
        CK(cudaGetDeviceProperties(&prop, dev));
        if (prop.major != 10 || prop.minor != 0)
            return set_err(SMLM_E_UNSUPPORTED, "device is not sm_100 (B200); this library is sm_100a-only");
        cached_dev = dev;
        cached_sms = prop.multiProcessorCount;
    }
    *num_sms = cached_sms;
    return SMLM_OK;
}

size_t smlm_adamw_workspace_size(void) {
    int sms = 0;
    if (current_sm100_sms(&sms) != SMLM_OK) return 0;
    return (size_t)sms * 8 * sizeof(float);
}

static int adamw_impl(float *param, float *exp_avg, float *exp_avg_sq, float *grad, int n_slots, size_t slot_stride,
                      int own_slot, void *param_bf16, size_t n, int step, float lr, float beta1, float beta2,
                      float eps, float weight_decay, float grad_scale, float max_grad_norm, int zero_grad,
                      const int *ready, int ready_target, void *ws, size_t ws_bytes, void *stream) {
    if (n == 0) return SMLM_OK;
    if (!param || !exp_avg || !exp_avg_sq || !grad) return set_err(SMLM_E_INVALID, "adamw: null buffer");
    if (step < 1) return set_err(SMLM_E_INVALID, "adamw: step must be >= 1");
    if (!(lr >= 0.f) || !(beta1 >= 0.f && beta1 < 1.f) || !(beta2 >= 0.f && beta2 < 1.f) || !(eps > 0.f) ||
        !(weight_decay >= 0.f) || !std::isfinite(grad_scale) || !std::isfinite(max_grad_norm))
        return set_err(SMLM_E_INVALID, "adamw: hyper-parameter out of range");
    if (n_slots < 1 || n_slots > kMaxRanks || own_slot < 0 || own_slot >= n_slots ||
        (n_slots > 1 && (slot_stride < n || slot_stride % 4)))
        return set_err(SMLM_E_INVALID, "adamw: 1 <= n_slots <= 8, 0 <= own_slot < n_slots, slot_stride >= n and a "
                                       "multiple of 4");
    auto al = [](const void *q, size_t b) { return (reinterpret_cast<uintptr_t>(q) % b) == 0; };
    if (!al(param, 16) || !al(exp_avg, 16) || !al(exp_avg_sq, 16) || !al(grad, 16) || (param_bf16 && !al(param_bf16, 8)))
        return set_err(SMLM_E_INVALID, "adamw: fp32 buffers must be 16-byte and the bf16 copy 8-byte aligned");
    int sms = 0, rc;
    if ((rc = current_sm100_sms(&sms))) return rc;
    cudaStream_t st = (cudaStream_t)stream;
    const int grid = adamw_grid(sms, n);
    AdamwArgs a;
    memset(&a, 0, sizeof(a));
    a.p = param;
    a.m = exp_avg;
    a.v = exp_avg_sq;
    a.g = grad;
    a.pb = reinterpret_cast<uint16_t *>(param_bf16);
    a.n = n;
    a.decay = (float)(1.0 - (double)lr * weight_decay);
    a.step_size = (float)((double)lr / (1.0 - std::pow((double)beta1, step)));
    a.inv_bc2_sqrt = (float)(1.0 / std::sqrt(1.0 - std::pow((double)beta2, step)));
    a.beta1 = beta1;
    a.beta2 = beta2;
    a.eps = eps;
    a.gscale = grad_scale;
    a.max_norm = max_grad_norm;
    a.zero_grad = zero_grad ? 1 : 0;
    a.partial = nullptr;
    a.n_partial = 0;
    a.n_slots = n_slots;
    a.slot_stride = n_slots > 1 ? slot_stride : 0;
    a.zero_slot = own_slot;
    a.ready = ready;
    a.ready_target = ready_target;
    if (max_grad_norm > 0.f) {
        if (!ws || !al(ws, 4) || ws_bytes < (size_t)grid * sizeof(float))
            return set_err(SMLM_E_WORKSPACE, "adamw: clipping needs smlm_adamw_workspace_size() bytes of workspace");
        ProfScope ps(4, st);
        CKL(launch_adamw_sumsq(a, reinterpret_cast<float *>(ws), grid, st), 1);
        a.partial = reinterpret_cast<const float *>(ws);
        a.n_partial = grid;
    }
    {
        ProfScope ps(4, st);
        CKL(launch_adamw_step(a, grid, st), 1);
    }
    return SMLM_OK;
}

int smlm_adamw_step(float *param, float *exp_avg, float *exp_avg_sq, float *grad, void *param_bf16, size_t n,
                    int step, float lr, float beta1, float beta2, float eps, float weight_decay, float grad_scale,
                    float max_grad_norm, int zero_grad, void *ws, size_t ws_bytes, void *stream) {
    return adamw_impl(param, exp_avg, exp_avg_sq, grad, 1, 0, 0, param_bf16, n, step, lr, beta1, beta2, eps,
                      weight_decay, grad_scale, max_grad_norm, zero_grad, nullptr, 0, ws, ws_bytes, stream);
}

int smlm_adamw_step_reduce(float *param, float *exp_avg, float *exp_avg_sq, float *grad_slots, int n_slots,
                           size_t slot_stride, int own_slot, void *param_bf16, size_t n, int step, float lr,
                           float beta1, float beta2, float eps, float weight_decay, float grad_scale,
                           float max_grad_norm, int zero_grad, const int *ready, int ready_target, void *ws,
                           size_t ws_bytes, void *stream) {
    return adamw_impl(param, exp_avg, exp_avg_sq, grad_slots, n_slots, slot_stride, own_slot, param_bf16, n, step, lr,
                      beta1, beta2, eps, weight_decay, grad_scale, max_grad_norm, zero_grad, ready, ready_target, ws,
                      ws_bytes, stream);
}

// ---- fused cross-rank reduction plumbing: IPC mappings, fan-out, completion ----
int smlm_ipc_get_handle(const void *dev_ptr, void *handle_out, uint64_t *offset_out) {
    if (!dev_ptr || !handle_out || !offset_out) return set_err(SMLM_E_INVALID, "NULL argument");
    // the handle names the whole allocation (e.g. a caching-allocator block): report ptr's offset
    static PFN_cuMemGetAddressRange_v3020 range = nullptr;
    if (!range) {
        void *fn = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuMemGetAddressRange", &fn, cudaEnableDefault, &q) != cudaSuccess || !fn)
            return set_err(SMLM_E_CUDA, "cuMemGetAddressRange entry point unavailable");
        range = reinterpret_cast<PFN_cuMemGetAddressRange_v3020>(fn);
    }
    CUdeviceptr base = 0;
    size_t size = 0;
    if (range(&base, &size, (CUdeviceptr)dev_ptr) != CUDA_SUCCESS)
        return set_err(SMLM_E_CUDA, "cuMemGetAddressRange failed");
    cudaIpcMemHandle_t h;
    CK(cudaIpcGetMemHandle(&h, reinterpret_cast<void *>(base)));
    static_assert(sizeof(h) == SMLM_IPC_HANDLE_BYTES, "IPC handle size");
    memcpy(handle_out, &h, sizeof(h));
    *offset_out = (uint64_t)((CUdeviceptr)dev_ptr - base);
    return SMLM_OK;
}

int smlm_ipc_open_handle(const void *handle, void **dev_ptr_out) {   // returns the allocation base
    if (!handle || !dev_ptr_out) return set_err(SMLM_E_INVALID, "NULL argument");
    cudaIpcMemHandle_t h;
    memcpy(&h, handle, sizeof(h));
    CK(cudaIpcOpenMemHandle(dev_ptr_out, h, cudaIpcMemLazyEnablePeerAccess));
    return SMLM_OK;
}

int smlm_ipc_close_handle(void *dev_ptr) {
    if (!dev_ptr) return SMLM_OK;
    CK(cudaIpcCloseMemHandle(dev_ptr));
    return SMLM_OK;
}

int smlm_pool_set_grad_fanout(smlm_pool p, int n_peers, const int64_t *byte_deltas) {
    if (!p) return set_err(SMLM_E_INVALID, "pool is NULL");
    if (n_peers < 0 || n_peers > kMaxRanks - 1 || (n_peers > 0 && !byte_deltas))
        return set_err(SMLM_E_INVALID, "fan-out: 0 <= n_peers <= 7 byte deltas");
    for (int q = 0; q < n_peers; ++q)
        if (byte_deltas[q] % 4) return set_err(SMLM_E_INVALID, "fan-out deltas must be multiples of 4 bytes");
    p->fanout.assign(byte_deltas, byte_deltas + n_peers);
    return SMLM_OK;
}

int smlm_fanout_signal(int n_ranks, int *const *ready_counters, void *stream) {
    if (n_ranks < 1 || n_ranks > kMaxRanks || !ready_counters) return set_err(SMLM_E_INVALID, "1 <= n_ranks <= 8");
    FanoutFlags f;
    memset(&f, 0, sizeof(f));
    f.n = n_ranks;
    for (int q = 0; q < n_ranks; ++q) {
        if (!ready_counters[q]) return set_err(SMLM_E_INVALID, "NULL ready counter");
        f.flag[q] = ready_counters[q];
    }
    CKL(launch_fanout_signal(f, (cudaStream_t)stream), 1);
    return SMLM_OK;
}

int smlm_fanout_wait(const int *ready, int target, void *stream) {
    if (!ready) return set_err(SMLM_E_INVALID, "NULL ready counter");
    CKL(launch_fanout_wait(ready, target, (cudaStream_t)stream), 1);
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
    if (e == cudaSuccess) e = cudaMemset(p->d_slots, 0, sizeof(SlotDev) * capacity);
    for (int i = 0; i < kCtrSets && e == cudaSuccess; ++i) {
        int *d = nullptr;
        e = cudaMalloc(&d, ctr_set_ints() * sizeof(int));
        if (e == cudaSuccess) {
            p->ctrs.push_back({(cudaStream_t)-1, d});
            e = cudaMemset(d, 0, ctr_set_ints() * sizeof(int));
        }
    }
    if (e != cudaSuccess) {
        cudaFree(p->d_slots);
        for (auto &c : p->ctrs) cudaFree(c.d);
        delete p;
        return cuda_err(e, "pool allocation");
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
        for (auto &c : p->ctrs) cudaFree(c.d);
        if (p->cap_arena) cudaFreeHost(p->cap_arena);
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
    if (option == SMLM_OPT_DECODE_KERNEL) {
        p->dec_kernel = value != 0;
        return SMLM_OK;
    }
    if (option == SMLM_OPT_DEC_COOPERATIVE) {
        p->dec_coop = value != 0;
        return SMLM_OK;
    }
    if (option == SMLM_OPT_DEC_KSPLIT) {
        if (value < 0 || value > 8) return set_err(SMLM_E_INVALID, "decode split-K must be in [0, 8]");
        p->dec_ksplit = value;
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
        d.r = h.r;
        if (p->dtype == SMLM_BF16) {
            // descriptors over the adapter's own rank: TMA zero-fills the rank indices past it, so
            // a lower-rank adapter is exactly the pool-rank one padded with zeros (f2)
            const int rb = p->r_pad * 2;
            int rc;
            if ((rc = make_map(&d.tmA, h.A, p->in, h.r, 64, p->r_pad, CU_TENSOR_MAP_SWIZZLE_128B))) return rc;
            // forward n-tile = 256 - r_pad output columns (the shrink rides in the same N=256 MMA)
            if ((rc = make_map(&d.tmBn, h.B, h.r, p->out, p->r_pad, 256 - p->r_pad, swizzle_for(rb)))) return rc;
            if ((rc = make_map(&d.tmBk, h.B, h.r, p->out, p->r_pad, 64, swizzle_for(rb)))) return rc;
        }
    }
    std::vector<uint8_t> bytes(sizeof(SlotDev));
    memcpy(bytes.data(), &d, sizeof(SlotDev));
    return stage_upload(p, bytes, p->d_slots + slot, st, true);
}

int smlm_adapter_register(smlm_pool p, const void *A, const void *B, float scale, void *stream, int *slot_out) {
    if (!p) return set_err(SMLM_E_INVALID, "NULL argument");
    return smlm_adapter_register_rank(p, A, B, p->r, scale, stream, slot_out);
}

int smlm_adapter_register_rank(smlm_pool p, const void *A, const void *B, int rank, float scale, void *stream,
                               int *slot_out) {
    if (!p || !A || !B || !slot_out) return set_err(SMLM_E_INVALID, "NULL argument");
    if (p->dtype == SMLM_BF16 ? (rank < 8 || rank > p->r || rank % 8 != 0) : rank != p->r)
        return set_err(SMLM_E_SHAPE, p->dtype == SMLM_BF16
                                         ? "adapter rank must be a multiple of 8 in [8, pool rank]"
                                         : "fp32 pools take adapters of the pool rank only");
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
    h.r = rank;
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
    const double h0 = g_hprof.on ? now_us() : 0;
    int rc = plan_for(p, b, false, plan);
    if (rc) return rc;
    if (b->S == 0 || b->G == 0) return SMLM_OK;
    if (!X || !Y) return set_err(SMLM_E_INVALID, "X and Y must be non-NULL");
    if (p->dtype == SMLM_BF16 && W) {
        // pure short / decode batch: one launch (kernels_dec3.cu)
        const double h1 = g_hprof.on ? now_us() : 0;
        const Dec3Plan D = dec3_plan(1, &p, b, plan);
        if (g_hprof.on) {
            g_hprof.t[0] += h1 - h0;
            g_hprof.t[1] += now_us() - h1;
            g_hprof.n++;
        }
        if (D.ok) {
            if (!ws || ws_bytes < D.total) return set_err(SMLM_E_WORKSPACE, "workspace too small");
            DeviceGuard dg(p->device);
            if ((rc = check_sticky())) return rc;
            return run_dec3(1, &p, b, D, X, &W, &Y, &V_save, reinterpret_cast<uint8_t *>(ws), (cudaStream_t)stream);
        }
    }
    const bool need_vf = p->dtype == SMLM_FP32;
    WsLayout L = layout_for(p, b, plan, false, need_vf);
    if (!ws || ws_bytes < L.total) return set_err(SMLM_E_WORKSPACE, "workspace too small");
    DeviceGuard dg(p->device);
    if ((rc = check_sticky())) return rc;
    cudaStream_t st = (cudaStream_t)stream;
    uint8_t *wsb = reinterpret_cast<uint8_t *>(ws);
    int *uctr = nullptr;
    if ((rc = stream_counters(p, st, nullptr, &uctr))) return rc;

    if (p->dtype == SMLM_FP32) {
        std::vector<uint8_t> bytes;
        append(bytes, plan.long_tiles);
        if ((rc = stage_upload(p, bytes, wsb + L.plan_off, st))) return rc;
        const DevTile *tiles = reinterpret_cast<const DevTile *>(wsb + L.plan_off);
        const int nt = (int)plan.long_tiles.size();
        float *Vf = reinterpret_cast<float *>(wsb + L.vf_off);
        CKL(launch_rows_shrink<float>(tiles, nt, p->d_slots, (const float *)X, p->in, p->r, Vf, (float *)V_save, 1,
                                      make_drop(b, p->in), st), 1);
        CKL(launch_f32_fwd(tiles, nt, p->d_slots, (const float *)X, (const float *)W, (float *)Y, Vf, p->in, p->out,
                           p->r, st), 1);
        return SMLM_OK;
    }

    // ---------------- bf16 tensor-core path ----------------
    if (b->dropout_p > 0.f && (!W || !p->cta_pair) && has_ft_lora(plan))
        return set_err(SMLM_E_UNSUPPORTED, "LoRA dropout on fine-tune rows needs W != NULL and SMLM_OPT_CTA_PAIR = 1 "
                                           "(the pre-shrink pass masks x; the fused 1-CTA shrink cannot)");
    FwdPrep F;
    if ((rc = fwd_prepare(p, b, plan, L, X, W, V_save, wsb, uctr, st, F))) return rc;
    if (F.n_tiles == 0) return SMLM_OK;
    if (F.pairs_dev) {
        __nv_bfloat16 *pre_sv = t_ext_pre_sv ? reinterpret_cast<__nv_bfloat16 *>(const_cast<void *>(t_ext_pre_sv))
                                             : reinterpret_cast<__nv_bfloat16 *>(wsb + L.pre_sv_off);
        if (F.n_pre_items && !t_ext_pre_sv) {
            // s*V = s X A_a^T once per long tile (split-K tensor-core contraction) -> tile-compact
            // bf16 + V_save; the CTA-pair GEMM then streams full 256-column W tiles
            ProfScope ps(2, st);
            UArgs u;
            memset(&u, 0, sizeof(u));
            if ((rc = make_map(&u.tmDY, X, p->in, b->S, 64, 128, CU_TENSOR_MAP_SWIZZLE_128B))) return rc;
            u.slots = p->d_slots;
            u.tiles = F.tiles_dev;
            u.items = F.pre_items_dev;
            u.n_items = F.n_pre_items;
            u.ksplit = L.pre_ksplit;
            u.K = p->in;
            u.r_pad = p->r_pad;
            u.part = reinterpret_cast<float *>(wsb + L.pre_part_off);
            u.sUt = pre_sv;
            u.vf = 1;
            u.r = p->r;
            u.Vsave = V_save;
            u.drop = make_drop(b, p->in);
            u.ctr = u.n_items <= kUCtrMax ? uctr : nullptr;
            CKL(launch_u(u, p->num_sms, st), u.ctr ? 1 : 2);
        }
        Gemm2Args g2;
        if ((rc = gemm2_fwd_args(1, &p, b, X, &W, &Y, &F, &pre_sv, g2))) return rc;
        ProfScope ps(0, st);
        CKL(launch_gemm2(g2, false, p->num_sms, st), 1);
        return SMLM_OK;
    }
    // one CTA per tile (SMLM_OPT_CTA_PAIR = 0, or W == NULL: Y holds the base output, LoRA term added)
    const bool has_w = W != nullptr;
    const int bnw = kBN - p->r_pad;
    GemmArgs a;
    memset(&a, 0, sizeof(a));
    if ((rc = make_map(&a.tmA, X, p->in, b->S, 64, 128, CU_TENSOR_MAP_SWIZZLE_128B))) return rc;
    if (has_w && (rc = make_map(&a.tmB, W, p->in, p->out, 64, bnw, CU_TENSOR_MAP_SWIZZLE_128B))) return rc;
    if (!plan.blocks.empty() &&
        (rc = make_map(&a.tmV, F.vbd, p->r_pad, plan.blocks.size() * 128, p->r_pad, 128, swizzle_for(p->r_pad * 2))))
        return rc;
    a.slots = p->d_slots;
    a.tiles = F.tiles_dev;
    a.blocks = F.blocks_dev;
    a.n_tiles = F.n_tiles;
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

// validate a multi-projection call; returns SMLM_OK and the plan of pools[0]
static int multi_check(int n_proj, const smlm_pool *pools, const smlm_batch *b, Plan &plan, bool &same_scales) {
    if (n_proj < 1 || n_proj > kDec3MaxProj) return set_err(SMLM_E_INVALID, "n_proj must be in [1, 4]");
    if (!pools || !b) return set_err(SMLM_E_INVALID, "NULL pools/batch");
    for (int i = 0; i < n_proj; ++i) {
        if (!pools[i]) return set_err(SMLM_E_INVALID, "NULL pool");
        if (pools[i]->device != pools[0]->device || pools[i]->in != pools[0]->in || pools[i]->r != pools[0]->r ||
            pools[i]->dtype != pools[0]->dtype)
            return set_err(SMLM_E_SHAPE, "pools must share device, in_features, rank and dtype");
    }
    int rc = plan_for(pools[0], b, false, plan);
    if (rc) return rc;
    same_scales = true;
    for (int g = 0; g < b->G; ++g) {
        const int sl = b->seg_slot[g];
        if (sl < 0) continue;
        for (int i = 1; i < n_proj; ++i) {
            if (sl >= pools[i]->cap || !pools[i]->ok[sl])
                return set_err(SMLM_E_SLOT, "slot " + std::to_string(sl) + " not registered in pool " + std::to_string(i));
            if (pools[i]->scales[sl] != pools[0]->scales[sl]) same_scales = false;
        }
    }
    return SMLM_OK;
}

// f1 for mixed batches: one pre-shrink pass over X for every projection (the A_a of all of them
// stacked as the N of one tcgen05 contraction), then each projection's GEMM with its s*V.
struct MultiPre {
    bool ok = false;
    bool merged = false;                  // all projections' GEMMs in ONE CTA-pair launch
    size_t base = 0;                      // per-projection forward workspace (max over pools)
    size_t base_off[kDec3MaxProj] = {};   // merged: one per projection (short-tile s*V live together)
    size_t sv_off[kDec3MaxProj] = {}, sv_bytes = 0;
    size_t part_off = 0, plan_off = 0, total = 0;
    int items = 0, ksplit = 1;
};
static MultiPre multi_pre_layout(int n_proj, const smlm_pool *pools, const smlm_batch *b, const Plan &plan, bool same) {
    MultiPre M;
    smlm_pool p0 = pools[0];
    if (!same || n_proj < 2 || p0->dtype != SMLM_BF16 || !use_preshrink(p0) ||
        n_proj * p0->r_pad > 128)
        return M;
    for (int i = 1; i < n_proj; ++i)
        if (pools[i]->cta_pair != p0->cta_pair || pools[i]->l_long != p0->l_long || pools[i]->r_pad != p0->r_pad)
            return M;
    for (auto &t : plan.long_tiles)
        if (t.slot >= 0) ++M.items;
    if (M.items == 0) return M;
    for (int i = 0; i < n_proj; ++i) M.base = std::max(M.base, smlm_workspace_size(pools[i], b, 0));
    M.merged = n_proj <= kGemm2MaxProj;
    size_t off = 0;
    for (int i = 0; i < (M.merged ? n_proj : 1); ++i) {
        M.base_off[i] = off;
        off = align256(off + M.base);
    }
    M.sv_bytes = plan.long_tiles.size() * 128 * (size_t)p0->r_pad * 2;
    for (int i = 0; i < n_proj; ++i) {
        M.sv_off[i] = off;
        off = align256(off + M.sv_bytes);
    }
    M.ksplit = u_ksplit(p0->num_sms, M.items, p0->in / 64);
    M.part_off = off;
    off = align256(off + (size_t)M.items * M.ksplit * 128 * n_proj * p0->r_pad * 4);
    M.plan_off = off;
    off = align256(off + plan.long_tiles.size() * sizeof(DevTile) + (size_t)M.items * sizeof(int) + 32);
    M.total = off;
    M.ok = true;
    return M;
}

size_t smlm_workspace_size_multi(int n_proj, const smlm_pool *pools, const smlm_batch *b) {
    Plan plan;
    bool same = true;
    if (multi_check(n_proj, pools, b, plan, same) != SMLM_OK) return 0;
    size_t ws = 0;
    for (int i = 0; i < n_proj; ++i) ws = std::max(ws, smlm_workspace_size(pools[i], b, 0));
    if (same) {
        const Dec3Plan D = dec3_plan(n_proj, pools, b, plan);
        if (D.ok) ws = std::max(ws, D.total);
    }
    const MultiPre M = multi_pre_layout(n_proj, pools, b, plan, same);
    if (M.ok) ws = std::max(ws, M.total);
    return ws;
}

int smlm_forward_multi(int n_proj, const smlm_pool *pools, const smlm_batch *b, const void *X, const void *const *W,
                       void *const *Y, void *const *V_save, void *ws, size_t ws_bytes, void *stream) {
    Plan plan;
    bool same = true;
    int rc = multi_check(n_proj, pools, b, plan, same);
    if (rc) return rc;
    if (b->S == 0 || b->G == 0) return SMLM_OK;
    if (!X || !W || !Y) return set_err(SMLM_E_INVALID, "X, W and Y must be non-NULL");
    for (int i = 0; i < n_proj; ++i)
        if (!W[i] || !Y[i]) return set_err(SMLM_E_INVALID, "W[i] and Y[i] must be non-NULL");
    if (b->dropout_p > 0.f && has_ft_lora(plan)) {
        // LoRA dropout: every projection draws its own mask (seed + i * golden), so the shared
        // pre-shrink cannot serve them all -- the per-projection calls
        for (int i = 0; i < n_proj; ++i) {
            const smlm_batch bi = batch_for_projection(b, i);
            if ((rc = smlm_forward(pools[i], &bi, X, W[i], Y[i], V_save ? V_save[i] : nullptr, ws, ws_bytes, stream)))
                return rc;
        }
        return SMLM_OK;
    }
    const Dec3Plan D = same ? dec3_plan(n_proj, pools, b, plan) : Dec3Plan();
    if (D.ok) {
        if (!ws || ws_bytes < D.total) return set_err(SMLM_E_WORKSPACE, "workspace too small");
        DeviceGuard dg(pools[0]->device);
        if ((rc = check_sticky())) return rc;
        return run_dec3(n_proj, pools, b, D, X, W, Y, V_save, reinterpret_cast<uint8_t *>(ws), (cudaStream_t)stream);
    }
    const MultiPre M = multi_pre_layout(n_proj, pools, b, plan, same);
    if (M.ok) {
        if (!ws || ws_bytes < M.total) return set_err(SMLM_E_WORKSPACE, "workspace too small");
        DeviceGuard dg(pools[0]->device);
        if ((rc = check_sticky())) return rc;
        smlm_pool p0 = pools[0];
        cudaStream_t st = (cudaStream_t)stream;
        uint8_t *wsb = reinterpret_cast<uint8_t *>(ws);
        int *uctr = nullptr;
        if ((rc = stream_counters(p0, st, nullptr, &uctr))) return rc;
        // long tiles (the same list every projection's forward builds) + the items with an adapter
        std::vector<int> items;
        for (size_t i = 0; i < plan.long_tiles.size(); ++i)
            if (plan.long_tiles[i].slot >= 0) items.push_back((int)i);
        std::vector<uint8_t> bytes;
        append(bytes, plan.long_tiles);
        while (bytes.size() % 16) bytes.push_back(0);
        const size_t items_off = bytes.size();
        append(bytes, items);
        if ((rc = stage_upload(p0, bytes, wsb + M.plan_off, st))) return rc;
        UArgs u;
        memset(&u, 0, sizeof(u));
        if ((rc = make_map_cached(p0, &u.tmDY, X, p0->in, b->S, 64, 128, CU_TENSOR_MAP_SWIZZLE_128B))) return rc;
        u.slots = p0->d_slots;
        u.tiles = reinterpret_cast<const DevTile *>(wsb + M.plan_off);
        u.items = reinterpret_cast<const int *>(wsb + M.plan_off + items_off);
        u.n_items = M.items;
        u.ksplit = M.ksplit;
        u.K = p0->in;
        u.r_pad = p0->r_pad;
        u.part = reinterpret_cast<float *>(wsb + M.part_off);
        u.vf = 1;
        u.r = p0->r;
        u.npj = n_proj;
        for (int i = 0; i < n_proj; ++i) {
            u.slots_p[i] = pools[i]->d_slots;
            u.sUt_p[i] = wsb + M.sv_off[i];
            u.Vsave_p[i] = V_save ? V_save[i] : nullptr;
        }
        u.ctr = u.n_items <= kUCtrMax ? uctr : nullptr;
        {
            ProfScope ps(2, st);
            CKL(launch_u(u, p0->num_sms, st), u.ctr ? 1 : 2);
        }
        if (!M.merged) {
            for (int i = 0; i < n_proj; ++i) {
                t_ext_pre_sv = wsb + M.sv_off[i];
                rc = smlm_forward(pools[i], b, X, W[i], Y[i], V_save ? V_save[i] : nullptr, ws, M.base, stream);
                t_ext_pre_sv = nullptr;
                if (rc) return rc;
            }
            return SMLM_OK;
        }
        // every projection's plan upload + short-row shrink in its own sub-workspace, then ONE
        // CTA-pair GEMM launch over the n-tiles of all projections (no per-projection wave tail)
        FwdPrep F[kGemm2MaxProj];
        __nv_bfloat16 *pre_sv[kGemm2MaxProj];
        for (int i = 0; i < n_proj; ++i) {
            const WsLayout Li = layout_for(pools[i], b, plan, false, false);
            if ((rc = fwd_prepare(pools[i], b, plan, Li, X, W[i], V_save ? V_save[i] : nullptr, wsb + M.base_off[i],
                                  uctr, st, F[i])))
                return rc;
            pre_sv[i] = reinterpret_cast<__nv_bfloat16 *>(wsb + M.sv_off[i]);
        }
        if (F[0].n_tiles == 0) return SMLM_OK;
        Gemm2Args g2;
        if ((rc = gemm2_fwd_args(n_proj, pools, b, X, W, Y, F, pre_sv, g2))) return rc;
        ProfScope ps(0, st);
        CKL(launch_gemm2(g2, false, p0->num_sms, st), 1);
        return SMLM_OK;
    }
    for (int i = 0; i < n_proj; ++i)
        if ((rc = smlm_forward(pools[i], b, X, W[i], Y[i], V_save ? V_save[i] : nullptr, ws, ws_bytes, stream)))
            return rc;
    return SMLM_OK;
}

// ---- backward phases (bf16 path; also the plan upload of the fp32 path) ----
struct BwdPrep {
    int nt = 0, n_pairs = 0, n_grad = 0, u_items = 0;
    const DevTile *tiles = nullptr;
    const void *groups = nullptr;
    const DevPair *pairs = nullptr;
    __nv_bfloat16 *sUt = nullptr, *sVt = nullptr;
    float *Uf = nullptr, *Vf = nullptr;
};

// grad groups + tiles + U items + CTA pairs -> workspace; bf16: the U pass (s*U, and s*V of the
// tile-compact dA/dB operand from V_save)
static int bwd_prepare(smlm_pool p, const smlm_batch *b, const Plan &plan, const WsLayout &L, const void *dY,
                       const void *V_save, bool want_dx, uint8_t *wsb, int *uctr, cudaStream_t st, BwdPrep &B) {
    int rc;
    // grad groups with the current grad bindings (masking: NULL => no dA/dB for that slot)
    std::vector<uint8_t> gbytes(plan.groups.size() * grad_group_bytes());
    int n_grad = 0;
    for (auto &g : plan.groups) {
        const SlotHost &h = p->slots[g.slot];
        if (!h.dA && !h.dB) continue;
        fill_grad_group(gbytes.data() + n_grad * grad_group_bytes(), g.slot, g.tile_begin, g.n_tiles, h.r, h.dA, h.dB);
        ++n_grad;
    }
    gbytes.resize(n_grad * grad_group_bytes());
    std::vector<int> uitems;
    for (size_t i = 0; i < plan.bwd_tiles.size(); ++i)
        if (plan.bwd_tiles[i].slot >= 0) uitems.push_back((int)i);
    // CTA pairs of consecutive fine-tune tiles (the dX GEMM on cta_group::2; any two tiles: a pair
    // of different adapters takes one expand block per adapter)
    std::vector<DevPair> bpairs;
    make_pairs(plan.bwd_tiles, bpairs);
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
    B.tiles = reinterpret_cast<const DevTile *>(wsb + L.plan_off);
    B.groups = wsb + L.plan_off + grp_off;
    B.pairs = reinterpret_cast<const DevPair *>(wsb + L.plan_off + bpair_off);
    B.n_pairs = (int)bpairs.size();
    B.nt = (int)plan.bwd_tiles.size();
    B.n_grad = n_grad;
    B.u_items = L.u_items;
    B.Uf = reinterpret_cast<float *>(wsb + L.u_off);
    B.Vf = reinterpret_cast<float *>(wsb + L.vf_off);
    B.sUt = reinterpret_cast<__nv_bfloat16 *>(wsb + L.sut_off);
    B.sVt = reinterpret_cast<__nv_bfloat16 *>(wsb + L.svt_off);
    if (p->dtype != SMLM_BF16) return SMLM_OK;
    // U = dY B_a per fine-tune tile (split-K tensor-core pass) -> tile-compact s*U
    if (L.u_items && (want_dx || n_grad)) {
        UArgs u;
        memset(&u, 0, sizeof(u));
        if ((rc = make_map(&u.tmDY, dY, p->out, b->S, 64, 128, CU_TENSOR_MAP_SWIZZLE_128B))) return rc;
        u.slots = p->d_slots;
        u.tiles = B.tiles;
        u.items = reinterpret_cast<const int *>(wsb + L.plan_off + uit_off);
        u.n_items = L.u_items;
        u.ksplit = L.u_ksplit;
        u.K = p->out;
        u.r_pad = p->r_pad;
        u.part = reinterpret_cast<float *>(wsb + L.upart_off);
        u.sUt = B.sUt;
        if (V_save && n_grad) {   // s*V folded into the reduce
            u.Vsave_in = V_save;
            u.sVt = B.sVt;
            u.r = p->r;
        }
        u.ctr = u.n_items <= kUCtrMax ? uctr : nullptr;
        CKL(launch_u(u, p->num_sms, st), u.ctr ? 1 : 2);
    }
    return SMLM_OK;
}

// the dX GEMM operands of one projection in a CTA-pair launch
static int bwd_gemm2_proj(smlm_pool p, const smlm_batch *b, const void *W, const void *dY, void *dX, const BwdPrep &B,
                          int nt0, Gemm2Proj &P) {
    int rc;
    if ((rc = make_map(&P.tmA, dY, p->out, b->S, 64, 128, CU_TENSOR_MAP_SWIZZLE_128B))) return rc;
    if ((rc = make_map(&P.tmW, W, p->in, p->out, 64, 64, CU_TENSOR_MAP_SWIZZLE_128B))) return rc;
    if (B.u_items) {
        if ((rc = make_map(&P.tmU, B.sUt, p->r_pad, (uint64_t)B.nt * 128, p->r_pad, 128, swizzle_for(p->r_pad * 2))))
            return rc;
        P.has_u = 1;
        P.u_rows = B.nt * 128;
    }
    P.slots = p->d_slots;
    P.Y = dX;
    P.N = p->in;
    P.K = p->out;
    P.nt0 = nt0;
    return SMLM_OK;
}

// dA/dB: the token contraction over the fine-tune tiles, per adapter in canonical order
static int bwd_tok(smlm_pool p, const smlm_batch *b, const void *X, const void *dY, const void *V_save,
                   int accumulate, const BwdPrep &B, cudaStream_t st) {
    int rc;
    if (!B.n_grad) return SMLM_OK;
    ProfScope ps(3, st);
    if (V_save) {
        if (!B.u_items)   // otherwise folded into the U pass
            CKL(launch_prep_sv<__nv_bfloat16>(B.tiles, B.nt, (const __nv_bfloat16 *)V_save, p->r, p->r_pad, B.sVt, st), 1);
    } else {
        CKL(launch_rows_shrink<__nv_bfloat16>(B.tiles, B.nt, p->d_slots, (const __nv_bfloat16 *)X, p->in, p->r, B.Vf,
                                              nullptr, 0, make_drop(b, p->in), st), 1);
        CKL(launch_prep_sv<float>(B.tiles, B.nt, B.Vf, p->r, p->r_pad, B.sVt, st), 1);
    }
    TokArgs ta;
    memset(&ta, 0, sizeof(ta));
    const int rb = p->r_pad * 2;
    if ((rc = make_map(&ta.tmX, X, p->in, b->S, 64, 64, CU_TENSOR_MAP_SWIZZLE_128B))) return rc;
    if ((rc = make_map(&ta.tmDY, dY, p->out, b->S, 64, 64, CU_TENSOR_MAP_SWIZZLE_128B))) return rc;
    if ((rc = make_map(&ta.tmSU, B.sUt, p->r_pad, (uint64_t)B.nt * 128, p->r_pad, 64, swizzle_for(rb)))) return rc;
    if ((rc = make_map(&ta.tmSV, B.sVt, p->r_pad, (uint64_t)B.nt * 128, p->r_pad, 64, swizzle_for(rb)))) return rc;
    ta.tiles = B.tiles;
    ta.groups = reinterpret_cast<const GradGroup *>(B.groups);
    ta.n_groups = B.n_grad;
    ta.in_f = p->in;
    ta.out_f = p->out;
    ta.r = p->r;
    ta.r_pad = p->r_pad;
    ta.nh = 2;   // 256-column items (two M=128 accumulators sharing the B operand)
    ta.mt_a = (p->in + 128 * ta.nh - 1) / (128 * ta.nh);
    ta.mt_b = (p->out + 128 * ta.nh - 1) / (128 * ta.nh);
    ta.accumulate = accumulate ? 1 : 0;
    ta.drop = make_drop(b, p->in);
    ta.n_fanout = (int)p->fanout.size();
    for (int q = 0; q < ta.n_fanout; ++q) ta.fanout_delta[q] = p->fanout[q];
    CKL(launch_tok(ta, p->num_sms, st), 1);
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
    int *uctr = nullptr;
    if ((rc = stream_counters(p, st, nullptr, &uctr))) return rc;
    BwdPrep B;
    if ((rc = bwd_prepare(p, b, plan, L, dY, V_save, dX != nullptr, wsb, uctr, st, B))) return rc;

    if (p->dtype == SMLM_FP32) {
        if (!p->fanout.empty() && B.n_grad)
            return set_err(SMLM_E_UNSUPPORTED, "gradient fan-out (smlm_pool_set_grad_fanout) is a bf16-path feature");
        CKL(launch_rows_u<float>(B.tiles, B.nt, p->d_slots, (const float *)dY, p->out, p->r, B.Uf, nullptr, p->r_pad,
                                 st), 1);
        const DropArgs drop = make_drop(b, p->in);
        if (dX)
            CKL(launch_f32_dx(B.tiles, B.nt, p->d_slots, (const float *)dY, (const float *)W, (float *)dX, B.Uf, p->in,
                              p->out, p->r, drop, st), 1);
        if (B.n_grad) {
            const float *V = (const float *)V_save;
            if (!V) {
                CKL(launch_rows_shrink<float>(B.tiles, B.nt, p->d_slots, (const float *)X, p->in, p->r, B.Vf, nullptr,
                                              0, drop, st), 1);
                V = B.Vf;
            }
            CKL((launch_dadb<float, float>(B.tiles, B.groups, B.n_grad, (const float *)X, (const float *)dY, B.Uf, V,
                                           p->in, p->out, p->r, accumulate, drop, st)), 2);
        }
        return SMLM_OK;
    }

    // ---------------- bf16 path ----------------
    if (dX) {
        ProfScope ps(1, st);
        if (p->cta_pair) {
            Gemm2Args g2;
            memset(&g2, 0, sizeof(g2));
            if ((rc = bwd_gemm2_proj(p, b, W, dY, dX, B, 0, g2.proj[0]))) return rc;
            g2.drop = make_drop(b, p->in);
            g2.pairs = B.pairs;
            g2.n_proj = 1;
            g2.n_pairs = B.n_pairs;
            g2.n_nt = (p->in + kBN - 1) / kBN;
            g2.group_m = (raster_group(p->out) + 1) / 2;
            g2.r = p->r;
            g2.r_pad = p->r_pad;
            g2.stages = gemm2_stages(p->r_pad);
            CKL(launch_gemm2(g2, true, p->num_sms, st), 1);
        } else {
            if (b->dropout_p > 0.f && B.u_items)
                return set_err(SMLM_E_UNSUPPORTED, "LoRA dropout needs SMLM_OPT_CTA_PAIR = 1 for dX (the mask multiplies "
                                                   "only the LoRA term: a separate accumulator)");
            GemmArgs a;
            memset(&a, 0, sizeof(a));
            if ((rc = make_map(&a.tmA, dY, p->out, b->S, 64, 128, CU_TENSOR_MAP_SWIZZLE_128B))) return rc;
            if ((rc = make_map(&a.tmB, W, p->in, p->out, 64, 64, CU_TENSOR_MAP_SWIZZLE_128B))) return rc;
            if (B.u_items && (rc = make_map(&a.tmV, B.sUt, p->r_pad, (uint64_t)B.nt * 128, p->r_pad, 128,
                                            swizzle_for(p->r_pad * 2))))
                return rc;
            a.slots = p->d_slots;
            a.tiles = B.tiles;
            a.blocks = nullptr;
            a.n_tiles = B.nt;
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
    return bwd_tok(p, b, X, dY, V_save, accumulate, B, st);
}

// ---- several projections that share X (q/k/v, gate/up): one dX GEMM launch ----
static int multi_bwd_check(int n_proj, const smlm_pool *pools, const smlm_batch *b, Plan &plan) {
    if (n_proj < 1 || n_proj > kGemm2MaxProj) return set_err(SMLM_E_INVALID, "n_proj must be in [1, 3]");
    if (!pools || !b) return set_err(SMLM_E_INVALID, "NULL pools/batch");
    for (int i = 0; i < n_proj; ++i) {
        if (!pools[i]) return set_err(SMLM_E_INVALID, "NULL pool");
        if (pools[i]->device != pools[0]->device || pools[i]->in != pools[0]->in || pools[i]->r != pools[0]->r ||
            pools[i]->dtype != pools[0]->dtype || pools[i]->cta_pair != pools[0]->cta_pair ||
            pools[i]->l_long != pools[0]->l_long)
            return set_err(SMLM_E_SHAPE, "pools must share device, in_features, rank, dtype and options");
    }
    for (int i = 0; i < n_proj; ++i) {
        Plan pl;
        int rc = plan_for(pools[i], b, true, i == 0 ? plan : pl);
        if (rc) return rc;
    }
    return SMLM_OK;
}

static size_t bwd_ws_each(int n_proj, const smlm_pool *pools, const smlm_batch *b, const Plan &plan, bool need_vf) {
    size_t m = 0;
    for (int i = 0; i < n_proj; ++i)
        m = std::max(m, layout_for(pools[i], b, plan, true, need_vf).total);
    return align256(m);
}

size_t smlm_workspace_size_backward_multi(int n_proj, const smlm_pool *pools, const smlm_batch *b) {
    Plan plan;
    if (multi_bwd_check(n_proj, pools, b, plan) != SMLM_OK) return 0;
    return (size_t)n_proj * bwd_ws_each(n_proj, pools, b, plan, true);
}

int smlm_backward_multi(int n_proj, const smlm_pool *pools, const smlm_batch *b, const void *X,
                        const void *const *W, const void *const *dY, const void *const *V_save, void *const *dX,
                        int accumulate, void *ws, size_t ws_bytes, void *stream) {
    Plan plan;
    int rc = multi_bwd_check(n_proj, pools, b, plan);
    if (rc) return rc;
    if (b->S == 0 || b->G == 0 || plan.bwd_tiles.empty()) return SMLM_OK;
    if (!X || !dY || !W || !dX) return set_err(SMLM_E_INVALID, "X, W, dY and dX arrays must be non-NULL");
    for (int i = 0; i < n_proj; ++i)
        if (!dY[i] || !W[i] || !dX[i]) return set_err(SMLM_E_INVALID, "W[i], dY[i] and dX[i] must be non-NULL");
    smlm_pool p0 = pools[0];
    const size_t each = bwd_ws_each(n_proj, pools, b, plan, true);
    if (!ws || ws_bytes < (size_t)n_proj * each) return set_err(SMLM_E_WORKSPACE, "workspace too small");
    const bool drop = b->dropout_p > 0.f && has_ft_lora(plan);
    if (p0->dtype != SMLM_BF16 || !p0->cta_pair || drop) {
        // one call per projection (same math; with LoRA dropout each projection has its own mask,
        // seed + i * golden, as smlm_forward_multi)
        for (int i = 0; i < n_proj; ++i) {
            const smlm_batch bi = batch_for_projection(b, i);
            if ((rc = smlm_backward(pools[i], &bi, X, W[i], dY[i], V_save ? V_save[i] : nullptr, dX[i], accumulate,
                                    reinterpret_cast<uint8_t *>(ws) + i * each, each, stream)))
                return rc;
        }
        return SMLM_OK;
    }
    DeviceGuard dg(p0->device);
    if ((rc = check_sticky())) return rc;
    cudaStream_t st = (cudaStream_t)stream;
    uint8_t *wsb = reinterpret_cast<uint8_t *>(ws);
    int *uctr = nullptr;
    if ((rc = stream_counters(p0, st, nullptr, &uctr))) return rc;
    BwdPrep B[kGemm2MaxProj];
    for (int i = 0; i < n_proj; ++i) {
        const void *vs = V_save ? V_save[i] : nullptr;
        Plan pl;
        if ((rc = plan_for(pools[i], b, true, pl))) return rc;
        const WsLayout L = layout_for(pools[i], b, pl, true, vs == nullptr);
        if ((rc = bwd_prepare(pools[i], b, pl, L, dY[i], vs, true, wsb + i * each, uctr, st, B[i]))) return rc;
    }
    {
        ProfScope ps(1, st);
        Gemm2Args g2;
        memset(&g2, 0, sizeof(g2));
        int nt0 = 0, kmax = 0;
        for (int i = 0; i < n_proj; ++i) {
            if ((rc = bwd_gemm2_proj(pools[i], b, W[i], dY[i], dX[i], B[i], nt0, g2.proj[i]))) return rc;
            nt0 += (pools[i]->in + kBN - 1) / kBN;
            kmax = std::max(kmax, pools[i]->out);
        }
        g2.pairs = B[0].pairs;
        g2.n_proj = n_proj;
        g2.n_pairs = B[0].n_pairs;
        g2.n_nt = nt0;
        g2.group_m = (raster_group(kmax) + 1) / 2;
        g2.r = p0->r;
        g2.r_pad = p0->r_pad;
        g2.stages = gemm2_stages(p0->r_pad);
        CKL(launch_gemm2(g2, true, p0->num_sms, st), 1);
    }
    for (int i = 0; i < n_proj; ++i)
        if ((rc = bwd_tok(pools[i], b, X, dY[i], V_save ? V_save[i] : nullptr, accumulate, B[i], st))) return rc;
    return SMLM_OK;
}

// ---- the Alg. 1 attention branch (kernels_attn.cu) ----
namespace {
struct AttnPlan {
    std::vector<AttnItem> items;
    std::vector<AttnRow> rows, drows;
    std::vector<AttnDGroup> dgroups;
    int max_dec_len = 0;
    int n_cache_rows = 0;   // PREFILL rows written to the cache
};
int attn_plan(const smlm_attn_batch *b, int n_heads, int n_kv_heads, int head_dim, int cache_slots, int capacity,
              AttnPlan &P) {
    if (!b) return set_err(SMLM_E_INVALID, "batch is NULL");
    if (head_dim != 128) return set_err(SMLM_E_UNSUPPORTED, "attention: head_dim must be 128");
    if (n_heads < 1 || n_kv_heads < 1 || n_heads % n_kv_heads ||
        (n_heads / n_kv_heads != 1 && n_heads / n_kv_heads != 2 && n_heads / n_kv_heads != 4 && n_heads / n_kv_heads != 8))
        return set_err(SMLM_E_SHAPE, "attention: n_heads must be 1, 2, 4 or 8 times n_kv_heads");
    if (b->S < 0 || b->G < 0 || (b->G > 0 && (!b->seg_offsets || !b->seg_mode)))
        return set_err(SMLM_E_INVALID, "attention: bad batch arrays");
    if (b->G == 0) return b->S == 0 ? SMLM_OK : set_err(SMLM_E_INVALID, "G == 0 but S != 0");
    const int32_t *off = b->seg_offsets;
    if (off[0] != 0 || off[b->G] != b->S) return set_err(SMLM_E_INVALID, "attention: offsets must run 0..S");
    for (int g = 0; g < b->G; ++g) {
        const int a0 = off[g], a1 = off[g + 1], L = a1 - a0, m = b->seg_mode[g];
        if (L < 0) return set_err(SMLM_E_INVALID, "attention: offsets must be non-decreasing");
        if (m < SMLM_FINETUNE || m > SMLM_DECODE) return set_err(SMLM_E_INVALID, "attention: mode outside 0..3");
        const int slot = b->seg_cache ? b->seg_cache[g] : -1;
        if (L == 0) continue;
        if (m == SMLM_DECODE) {
            const int past = b->seg_past ? b->seg_past[g] : 0;
            if (slot < 0 || slot >= cache_slots || past < 0 || past + L > capacity)
                return set_err(SMLM_E_INVALID, "attention: a DECODE segment needs a cache slot with room for its rows");
            // groups of up to kAttnDecCols / G rows share one read of the slot's K / V
            const int rg = kAttnDecCols / (n_heads / n_kv_heads);
            for (int i = 0; i < L; ++i) {
                if (i % rg == 0) P.dgroups.push_back({(int)P.drows.size(), std::min(rg, L - i), past + i, slot});
                // appended to the cache by the decode kernel; pad = the segment's first new position
                P.drows.push_back({a0 + i, slot, past + i, past});
            }
            P.max_dec_len = std::max(P.max_dec_len, past + L);
        } else {
            if (m == SMLM_PREFILL && slot >= 0) {
                if (slot >= cache_slots || L > capacity)
                    return set_err(SMLM_E_INVALID, "attention: PREFILL cache slot out of range or too short");
                // one cache-write record per segment {first row, slot, rows before it in the
                // write list, length}: a small plan (the parameter-blob upload, not a memcpy)
                P.rows.push_back({a0, slot, P.n_cache_rows, L});
                P.n_cache_rows += L;
            }
            for (int qb = 0; qb * 128 < L; ++qb) P.items.push_back({a0, L, qb, 0});
        }
    }
    // the longest items (most key blocks) first: the persistent CTAs finish together
    std::stable_sort(P.items.begin(), P.items.end(), [](const AttnItem &x, const AttnItem &y) { return x.qb > y.qb; });
    return SMLM_OK;
}
smlm_pool_s g_attn_stage;   // pinned staging of the attention plans (no adapter pool involved)
}  // namespace

static size_t attn_plan_bytes(const AttnPlan &P) {
    return align256(P.items.size() * sizeof(AttnItem) + P.rows.size() * sizeof(AttnRow) +
                    P.drows.size() * sizeof(AttnRow) + P.dgroups.size() * sizeof(AttnDGroup) + 64);
}
static size_t attn_part_bytes(const AttnPlan &P, int n_heads, int n_kv_heads) {
    const size_t splits = (size_t)(P.max_dec_len + kAttnDecChunk - 1) / kAttnDecChunk;
    return align256(P.drows.size() * (size_t)n_heads * splits * 130 * sizeof(float));
}

size_t smlm_attention_workspace_size(const smlm_attn_batch *b, int n_heads, int n_kv_heads) {
    if (!b || n_heads < 1 || n_kv_heads < 1) return 0;
    AttnPlan P;
    if (attn_plan(b, n_heads, n_kv_heads, 128, 1 << 30, 1 << 30, P) != SMLM_OK) return 0;
    return attn_plan_bytes(P) + attn_part_bytes(P, n_heads, n_kv_heads) + 256;
}

int smlm_attention(const smlm_attn_batch *b, int n_heads, int n_kv_heads, int head_dim, const void *Q, const void *K,
                   const void *V, void *O, void *K_cache, void *V_cache, int cache_slots, int cache_capacity,
                   float scale, void *ws, size_t ws_bytes, void *stream) {
    AttnPlan P;
    int rc = attn_plan(b, n_heads, n_kv_heads, head_dim, cache_slots, cache_capacity, P);
    if (rc) return rc;
    if (b->S == 0) return SMLM_OK;
    if (!Q || !K || !V || !O) return set_err(SMLM_E_INVALID, "attention: Q, K, V and O must be non-NULL");
    if ((!P.rows.empty() || !P.drows.empty()) && (!K_cache || !V_cache))
        return set_err(SMLM_E_INVALID, "attention: prefill-with-cache / decode segments need K_cache and V_cache");
    if (!(scale > 0.f) || !std::isfinite(scale)) return set_err(SMLM_E_INVALID, "attention: scale must be finite, > 0");
    const size_t need = attn_plan_bytes(P) + attn_part_bytes(P, n_heads, n_kv_heads) + 256;
    if (!ws || ws_bytes < need) return set_err(SMLM_E_WORKSPACE, "workspace too small");
    int sms = 0;
    if ((rc = current_sm100_sms(&sms))) return rc;
    if ((rc = check_sticky())) return rc;
    cudaStream_t st = (cudaStream_t)stream;
    uint8_t *wsb = reinterpret_cast<uint8_t *>(ws);
    std::vector<uint8_t> bytes;
    append(bytes, P.items);
    while (bytes.size() % 16) bytes.push_back(0);
    const size_t rows_off = bytes.size();
    append(bytes, P.rows);
    const size_t drows_off = bytes.size();
    append(bytes, P.drows);
    const size_t dgroups_off = bytes.size();
    append(bytes, P.dgroups);
    // a small decode plan rides in the decode kernels' parameters; nothing to upload for a
    // decode-only call then
    const bool dec_inline = P.drows.size() <= (size_t)kAttnDecInline && P.dgroups.size() <= (size_t)kAttnDecInline;
    static thread_local AttnDecInline dinl;
    if (dec_inline) {
        std::copy(P.drows.begin(), P.drows.end(), dinl.drows);
        std::copy(P.dgroups.begin(), P.dgroups.end(), dinl.dgroups);
    }
    const bool upload = !(dec_inline && P.items.empty() && P.rows.empty());
    if (upload && (rc = stage_upload(&g_attn_stage, bytes, wsb, st))) return rc;
    AttnArgs a;
    memset(&a, 0, sizeof(a));
    a.dbg = measure_flag("SMLM_ATTN_DEBUG");
    const uint64_t S = (uint64_t)b->S;
    if (!P.items.empty()) {
        if ((rc = make_map(&a.tmQ, Q, (uint64_t)n_heads * 128, S, 64, 128, CU_TENSOR_MAP_SWIZZLE_128B))) return rc;
        if ((rc = make_map(&a.tmK, K, (uint64_t)n_kv_heads * 128, S, 64, 128, CU_TENSOR_MAP_SWIZZLE_128B))) return rc;
        if ((rc = make_map(&a.tmV, V, (uint64_t)n_kv_heads * 128, S, 64, 64, CU_TENSOR_MAP_SWIZZLE_128B))) return rc;
        if ((rc = make_map(&a.tmO, O, (uint64_t)n_heads * 128, S, 64, 128, CU_TENSOR_MAP_SWIZZLE_128B))) return rc;
    }
    if (!P.drows.empty()) {
        const uint64_t crow = (uint64_t)cache_slots * (uint64_t)cache_capacity;
        if ((rc = make_map(&a.tmKc, K_cache, (uint64_t)n_kv_heads * 128, crow, 64, 128, CU_TENSOR_MAP_SWIZZLE_128B))) return rc;
        if ((rc = make_map(&a.tmVc, V_cache, (uint64_t)n_kv_heads * 128, crow, 64, 128, CU_TENSOR_MAP_SWIZZLE_128B))) return rc;
    }
    a.items = reinterpret_cast<const AttnItem *>(wsb);
    a.rows = reinterpret_cast<const AttnRow *>(wsb + rows_off);
    a.drows = reinterpret_cast<const AttnRow *>(wsb + drows_off);
    a.dgroups = reinterpret_cast<const AttnDGroup *>(wsb + dgroups_off);
    a.Q = Q;
    a.K = K;
    a.V = V;
    a.O = O;
    a.K_cache = K_cache;
    a.V_cache = V_cache;
    a.n_heads = n_heads;
    a.n_kv_heads = n_kv_heads;
    a.cache_capacity = cache_capacity;
    a.scale = scale;
    a.max_splits = (P.max_dec_len + kAttnDecChunk - 1) / kAttnDecChunk;
    a.dpart = reinterpret_cast<float *>(wsb + attn_plan_bytes(P));
    // launches: the cache write of PREFILL rows, the prefill kernel, the decode split + combine
    const bool fused_rows = !P.items.empty() && (n_heads / n_kv_heads) % 2 == 0 && n_kv_heads <= 8;   // prefill warp 2
    const int nl = (P.rows.empty() || fused_rows ? 0 : 1) + (P.items.empty() ? 0 : 1) + (P.drows.empty() ? 0 : 2);
    a.dec_inline = dec_inline ? 1 : 0;
    a.n_rows = (int)P.rows.size();
    a.n_cache_rows = P.n_cache_rows;
    CKL(launch_attn(a, dinl, (int)P.items.size(), (int)P.rows.size(), (int)P.drows.size(), (int)P.dgroups.size(), st), nl);
    return SMLM_OK;
}

}  // extern "C"
