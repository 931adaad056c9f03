// runtime.cuh -- host orchestration of the kernels (included by capi.cu and the per-parameter-set
// translation units ps_<p>.cu; split so the six parameter sets compile in parallel).
#pragma once
//
// BatchKeyGen (Algorithm 1) per chunk of keys, all on one stream:
//   sample (f, g + small-factor isInvertible, retries)          sample.cuh
//   R/3 batchInv: product-tree up-sweep, root divstep, down-sweep, repair of failed trees
//   R/q batchInv on [3f]: up-sweep, root divstep, down-sweep     ringmul.cuh, divstep.cuh
//   H = [g * fbar]                                                ringmul.cuh (ZIP)
//   encode pk, sk                                                 encode.cuh
// batchInv is Montgomery's trick arranged as a tree: level l multiplies sibling
// pairs (cnt_l = ceil(cnt_{l-1}/2) products), one inversion per tree root, then each child's
// inverse = parent inverse * sibling: 3(B-1) products per full tree of B leaves, as the
// paper's chain.
#include <atomic>
#include <cmath>
#include <cstdlib>
#include <cstdio>
#include <cstring>
#include <map>
#include <tuple>
#include <mutex>
#include <string>
#include <vector>

#include "../../include/sntrup_gpu.h"
#include "common.cuh"
#include "divstep.cuh"
#include "jump.cuh"
#include "encode.cuh"
#include "factor_tables.h"
#include "fullsk.cuh"
#include "intpeak.cuh"
#include "ringmul.cuh"
#include "sample.cuh"
#include "tcmul.cuh"
#include "tc4mul.cuh"
#include "tc4w.cuh"
#include "tcxmul.cuh"


namespace sntrup_rt {
using namespace sntrup;

inline std::atomic<uint64_t> g_launches{0};
inline std::mutex g_mu;                                   // serialises calls (shared workspace)

// ------------------------------------------------------------------------------ profiler
// Optional per-launch CUDA-event timing on the launching stream (bench.py's roofline): every
// launch of kernel class k records (start, end) events and `units` of work (products, keys,
// inversions).  Read back with sntrup_profile_read().
enum ProfClass { PC_SAMPLE = 0, PC_MUL_R3, PC_MUL_RQ, PC_INV_R3, PC_INV_RQ, PC_REPAIR, PC_ENCODE,
                 PC_MISC, PC_N };
struct ProfRec { int cls; cudaEvent_t a, b; double units, ops; int kind; double smem; cudaStream_t s; };
inline bool g_prof_on = false;
inline std::vector<ProfRec> g_prof;
inline std::vector<cudaEvent_t> g_evpool;
struct ProfAgg { double ms = 0, units = 0, ops = 0, smem = 0; uint64_t launches = 0; };
inline ProfAgg g_agg[PC_N];
// ring-product launches by arithmetic kind: 0 = int8 tensor (kind::i8), 1 = fp4 tensor
// (kind::mxf4), 2 = int32 schoolbook
enum { PK_I8 = 0, PK_F4 = 1, PK_I32 = 2, PK_N = 3 };
inline ProfAgg g_kagg[PK_N];
inline int g_cur_kind = -1;                 // set by the launcher inside a ProfScope
inline double g_cur_smem = 0;               // tensor-core operand bytes the launch's MMAs fetch from smem

inline cudaEvent_t ev_get() {
    if (!g_evpool.empty()) { cudaEvent_t e = g_evpool.back(); g_evpool.pop_back(); return e; }
    cudaEvent_t e;
    cudaEventCreate(&e);
    return e;
}

struct ProfScope {
    int cls; double units, ops; cudaStream_t s; cudaEvent_t a = nullptr;
    // units: products / keys / inversions; ops: algorithmic integer ops of the launch (0 if n/a)
    ProfScope(int c, double u, cudaStream_t st, double o = 0) : cls(c), units(u), ops(o), s(st) {
        if (g_prof_on) { a = ev_get(); cudaEventRecord(a, s); }
    }
    ~ProfScope() {
        if (a) { cudaEvent_t b = ev_get(); cudaEventRecord(b, s); g_prof.push_back(ProfRec{cls, a, b, units, ops, g_cur_kind, g_cur_smem, s}); }
        g_cur_kind = -1;
        g_cur_smem = 0;
    }
};

inline void prof_drain() {
    // SNTRUP_TIMELINE=<file> (diagnostic): append one line per launch -- class, arithmetic kind,
    // units, stream, and the times (ms, from the drain's first record) at which the launch became
    // runnable on its stream (start event) and finished (end event); scripts/timeline.py
    FILE *tl = nullptr;
    if (!g_prof.empty()) {
        const char *tp = getenv("SNTRUP_TIMELINE");
        if (tp && *tp) tl = fopen(tp, "a");
    }
    for (auto &r : g_prof) {
        cudaEventSynchronize(r.b);
        float ms = 0;
        cudaEventElapsedTime(&ms, r.a, r.b);
        if (tl) {
            float t0 = 0;
            cudaEventSynchronize(g_prof.front().a);
            cudaEventElapsedTime(&t0, g_prof.front().a, r.a);
            fprintf(tl, "%d,%d,%.0f,%llx,%.4f,%.4f\n", r.cls, r.kind, r.units, (unsigned long long)(uintptr_t)r.s,
                    t0, t0 + ms);
        }
        g_agg[r.cls].ms += ms;
        g_agg[r.cls].units += r.units;
        g_agg[r.cls].ops += r.ops;
        if (r.kind >= 0) {
            g_kagg[r.kind].ms += ms;
            g_kagg[r.kind].ops += r.ops;
            g_kagg[r.kind].units += r.units;
            g_kagg[r.kind].smem += r.smem;
            g_kagg[r.kind].launches += 1;
        }
        g_agg[r.cls].launches += 1;
        g_evpool.push_back(r.a);
        g_evpool.push_back(r.b);
    }
    if (tl) { fprintf(tl, "#\n"); fclose(tl); }
    g_prof.clear();
}

#define CK(x)                                                                      \
    do {                                                                           \
        cudaError_t e_ = (x);                                                      \
        if (e_ != cudaSuccess) {                                                   \
            fprintf(stderr, "sntrup_gpu: %s failed: %s (%s:%d)\n", #x,             \
                    cudaGetErrorString(e_), __FILE__, __LINE__);                   \
            return SNTRUP_E_CUDA;                                                  \
        }                                                                          \
    } while (0)

#define LAUNCHED()                                                                 \
    do {                                                                           \
        g_launches.fetch_add(1, std::memory_order_relaxed);                        \
        cudaError_t e_ = cudaGetLastError();                                       \
        if (e_ != cudaSuccess) {                                                   \
            fprintf(stderr, "sntrup_gpu: launch failed: %s (%s:%d)\n",             \
                    cudaGetErrorString(e_), __FILE__, __LINE__);                   \
            return SNTRUP_E_CUDA;                                                  \
        }                                                                          \
    } while (0)

// ------------------------------------------------------------------------------ param info
struct ParamInfo { int p, q, w, p16, p8; size_t pk, sk; };

inline size_t rq_encoded_len(int p, int q) {
    std::vector<uint32_t> M(p, (uint32_t)q);
    size_t len = 0;
    int n = p;
    while (n > 1) {
        std::vector<uint32_t> M2((n + 1) / 2);
        for (int i = 0; i + 1 < n; i += 2) {
            uint32_t m = M[i] * M[i + 1];
            while (m >= 16384u) { len++; m = (m + 255u) >> 8; }
            M2[i / 2] = m;
        }
        if (n & 1) M2[n / 2] = M[n - 1];
        M.swap(M2);
        n = (n + 1) / 2;
    }
    uint32_t m = M[0];
    while (m > 1) { len++; m = (m + 255u) >> 8; }
    return len;
}

inline bool param_info(int ps, ParamInfo *pi) {
    static const int tab[][3] = {{653, 4621, 288}, {761, 4591, 286}, {857, 5167, 322},
                                 {953, 6343, 396}, {1013, 7177, 448}, {1277, 7879, 492}};
    for (auto &t : tab)
        if (t[0] == ps) {
            pi->p = t[0]; pi->q = t[1]; pi->w = t[2];
            pi->p16 = (t[0] + 15) / 16 * 16;
            pi->p8 = (t[0] + 7) / 8 * 8;
            pi->pk = rq_encoded_len(t[0], t[1]);
            pi->sk = 2 * (size_t)((t[0] + 3) / 4);
            return true;
        }
    return false;
}

// ------------------------------------------------------------------------------ device tables
struct DevTables {
    uint2 *T = nullptr;          // [P][WT] small-factor residues of x^j
    uint32_t *masks = nullptr;   // [nf][WT]
    int nf = 0, wt = 0;
    uint32_t *Mlo = nullptr;
    uint8_t *emit = nullptr;
    uint16_t *off = nullptr;
    EncTables enc{};
    double p_small_reject = 0;   // 1 - prod (1 - 3^-d) over the small factors' degrees d
};
inline std::map<std::pair<int, int>, DevTables> g_tables;    // (device, param) -> tables

inline int build_tables(int dev, int ps, int WT, DevTables **out) {
    auto key = std::make_pair(dev, ps);
    auto it = g_tables.find(key);
    if (it != g_tables.end()) { *out = &it->second; return SNTRUP_OK; }
    ParamInfo pi;
    param_info(ps, &pi);
    const int p = pi.p;
    DevTables t;
    // -- small-factor residue table: row j = concat_i (x^j mod f_i), bitsliced
    const sntrup_tables::SmallFactorSet *fs = nullptr;
    for (auto &s : sntrup_tables::kSmallFactors) if (s.p == p) fs = &s;
    if (!fs) return SNTRUP_E_PARAM;
    int S = 0;
    for (int i = 0; i < fs->count; i++) S += fs->deg[i];
    const int wt = (S + 31) / 32;
    if (wt != WT) { fprintf(stderr, "sntrup_gpu: factor table width mismatch\n"); return SNTRUP_E_PARAM; }
    std::vector<uint2> T((size_t)p * WT, make_uint2(0, 0));
    std::vector<uint32_t> masks((size_t)fs->count * WT, 0);
    int o = 0;
    for (int fi = 0; fi < fs->count; fi++) {
        const int d = fs->deg[fi];
        std::vector<int> f(d + 1), r(d, 0);
        for (int i = 0; i <= d; i++) f[i] = fs->coef[fi][i] - '0';
        r[0] = 1 % 3;
        for (int j = 0; j < p; j++) {
            for (int i = 0; i < d; i++) {
                const int pos = o + i, w = pos / 32, bit = pos % 32;
                if (r[i] == 1) T[(size_t)j * WT + w].x |= 1u << bit;
                if (r[i] == 2) T[(size_t)j * WT + w].y |= 1u << bit;
            }
            // r <- x * r mod f (f monic of degree d)
            const int top = r[d - 1];
            for (int i = d - 1; i > 0; i--) r[i] = r[i - 1];
            r[0] = 0;
            for (int i = 0; i < d; i++) r[i] = ((r[i] - top * f[i]) % 3 + 3) % 3;
        }
        for (int i = 0; i < d; i++) masks[(size_t)fi * WT + (o + i) / 32] |= 1u << ((o + i) % 32);
        o += d;
    }
    t.nf = fs->count;
    t.wt = WT;
    {
        double keep = 1.0;
        for (int fi = 0; fi < fs->count; fi++) keep *= 1.0 - std::pow(3.0, -fs->deg[fi]);
        t.p_small_reject = 1.0 - keep;
    }
    // -- encode tables (C10): per level, per pair (M_{2i}, bytes, offset)
    std::vector<uint32_t> Mlo;
    std::vector<uint8_t> emit;
    std::vector<uint16_t> off;
    EncTables enc{};
    {
        std::vector<uint32_t> M(p, (uint32_t)pi.q);
        int n = p, lev = 0;
        uint32_t pos = 0;
        while (n > 1) {
            if (lev >= ENC_MAXLEV) return SNTRUP_E_PARAM;
            enc.lev_n[lev] = n;
            enc.lev_pair_base[lev] = (int)Mlo.size();
            enc.lev_off[lev] = (int)pos;
            std::vector<uint32_t> M2((n + 1) / 2);
            for (int i = 0; i + 1 < n; i += 2) {
                uint32_t m = M[i] * M[i + 1];
                int e = 0;
                while (m >= 16384u) { e++; m = (m + 255u) >> 8; }
                Mlo.push_back(M[i]);
                emit.push_back((uint8_t)e);
                off.push_back((uint16_t)pos);
                pos += e;
                M2[i / 2] = m;
            }
            if (n & 1) M2[n / 2] = M[n - 1];
            M.swap(M2);
            n = (n + 1) / 2;
            lev++;
        }
        enc.nlev = lev;
        // per-level uniform form used by the kernel (checked here)
        for (int l = 0; l < lev; l++) {
            const int base = enc.lev_pair_base[l], np = enc.lev_n[l] / 2;
            enc.lev_M[l] = Mlo[base];
            enc.lev_e[l] = emit[base];
            enc.lev_elast[l] = emit[base + np - 1];
            for (int i = 0; i < np; i++) {
                if (Mlo[base + i] != enc.lev_M[l]) return SNTRUP_E_INTERNAL;
                if (i < np - 1 && emit[base + i] != enc.lev_e[l]) return SNTRUP_E_INTERNAL;
                if (off[base + i] != enc.lev_off[l] + enc.lev_e[l] * i) return SNTRUP_E_INTERNAL;
            }
        }
        uint32_t m = M[0];
        int e = 0;
        while (m > 1) { e++; m = (m + 255u) >> 8; }
        enc.top_emit = e;
        enc.top_off = (int)pos;
        enc.pk_bytes = (int)(pos + e);
        if ((size_t)enc.pk_bytes != pi.pk) return SNTRUP_E_INTERNAL;
        // the kernel's compile-time plan must be this table
        bool same = false;
        auto cmp = [&](const EncPlan &c) {
            same = c.nlev == enc.nlev && c.top_emit == enc.top_emit && c.top_off == enc.top_off &&
                   c.pk_bytes == enc.pk_bytes;
            for (int l = 0; same && l < enc.nlev; l++)
                same = c.lev_n[l] == enc.lev_n[l] && c.lev_e[l] == enc.lev_e[l] &&
                       c.lev_elast[l] == enc.lev_elast[l] && c.lev_off[l] == enc.lev_off[l] &&
                       c.lev_M[l] == enc.lev_M[l];
            return 0;
        };
        SNTRUP_DISPATCH(p, cmp(EncPlanOf<PS>::v));
        if (!same) return SNTRUP_E_INTERNAL;
    }
    CK(cudaMalloc(&t.T, T.size() * sizeof(uint2)));
    CK(cudaMemcpy(t.T, T.data(), T.size() * sizeof(uint2), cudaMemcpyHostToDevice));
    CK(cudaMalloc(&t.masks, masks.size() * sizeof(uint32_t)));
    CK(cudaMemcpy(t.masks, masks.data(), masks.size() * sizeof(uint32_t), cudaMemcpyHostToDevice));
    CK(cudaMalloc(&t.Mlo, Mlo.size() * sizeof(uint32_t)));
    CK(cudaMemcpy(t.Mlo, Mlo.data(), Mlo.size() * sizeof(uint32_t), cudaMemcpyHostToDevice));
    CK(cudaMalloc(&t.emit, emit.size()));
    CK(cudaMemcpy(t.emit, emit.data(), emit.size(), cudaMemcpyHostToDevice));
    CK(cudaMalloc(&t.off, off.size() * sizeof(uint16_t)));
    CK(cudaMemcpy(t.off, off.data(), off.size() * sizeof(uint16_t), cudaMemcpyHostToDevice));
    enc.Mlo = t.Mlo;
    enc.emit = t.emit;
    enc.off = t.off;
    t.enc = enc;
    auto res = g_tables.emplace(key, t);
    *out = &res.first->second;
    return SNTRUP_OK;
}

// ------------------------------------------------------------------------------ copy stream
// Host-output keygen: chunk i's pk/sk are copied device->host on a copy stream while chunk i+1
// computes (double-buffered device staging).  One per device (calls are serialised).
struct CopyStream { cudaStream_t s = nullptr; cudaEvent_t comp[2] = {}, copy[2] = {}; };
inline std::vector<cudaStream_t> g_copy_streams;     // every copy stream created (staging layout changes)
// SNTRUP_OPT_LANE_PRIORITY: lane li's streams get priority rank li (lane 0 highest), so the
// scheduler finishes lane 0's chunk first while the other lanes fill its latency gaps; -1 = the
// default priority.
inline int lane_priority(int prio_rank) {
    if (prio_rank < 0) return 0;
    int least = 0, greatest = 0;
    cudaDeviceGetStreamPriorityRange(&least, &greatest);
    const int p = greatest + prio_rank;                  // greatest is numerically lowest
    return p > least ? least : p;
}

inline int make_stream(cudaStream_t *s, int prio_rank) {
    if (prio_rank < 0) CK(cudaStreamCreateWithFlags(s, cudaStreamNonBlocking));
    else CK(cudaStreamCreateWithPriority(s, cudaStreamNonBlocking, lane_priority(prio_rank)));
    return SNTRUP_OK;
}

// ------------------------------------------------------------------------------ tree-top routing
// Inside a bulk keygen call the tree tops (levels of a few hundred work items) and the root
// inversions are a chain of small, latency-bound launches.  On the lane's own stream they queue
// behind the other lane's bulk kernels, whose persistent CTAs hold every shared-memory slot of the
// SMs until their launch ends.  With routing on (sntrup_set_sched: top_items > 0), a launch of
// <= top_items work items goes to a high-priority companion stream of its chain (ordered with the
// chain by an event at every switch), and with items_cap > 0 a bulk launch's grid grows to
// ceil(items / items_cap) CTAs, so CTAs retire after items_cap items and the block scheduler
// hands the freed slot to a waiting high-priority CTA first.
struct TopRoute { cudaStream_t hi = nullptr; cudaEvent_t ev = nullptr; bool on_hi = false; };
inline bool g_route_on = false;             // set for the duration of a bulk keygen call
inline long long g_top_items = 0;           // sntrup_set_sched
inline long long g_items_cap = 0;
inline std::map<std::pair<int, uintptr_t>, TopRoute> g_routes;

inline int route_stream(cudaStream_t s, bool top, cudaStream_t *out) {
    *out = s;
    if (!g_route_on) return SNTRUP_OK;
    int dev = 0;
    CK(cudaGetDevice(&dev));
    TopRoute &r = g_routes[std::make_pair(dev, (uintptr_t)s)];
    if (!r.hi) {
        if (!top) return SNTRUP_OK;
        CK(cudaStreamCreateWithPriority(&r.hi, cudaStreamNonBlocking, lane_priority(0)));
        CK(cudaEventCreateWithFlags(&r.ev, cudaEventDisableTiming));
    }
    if (top != r.on_hi) {
        CK(cudaEventRecord(r.ev, r.on_hi ? r.hi : s));
        CK(cudaStreamWaitEvent(r.on_hi ? s : r.hi, r.ev, 0));
        r.on_hi = top;
    }
    *out = top ? r.hi : s;
    return SNTRUP_OK;
}
// back onto the chain's own stream (before anything but a ring product / root launch touches it)
inline int route_flush(cudaStream_t s) {
    cudaStream_t t;
    return route_stream(s, false, &t);
}
inline bool stream_capturing(cudaStream_t s) {
    cudaStreamCaptureStatus st = cudaStreamCaptureStatusNone;
    return cudaStreamIsCapturing(s, &st) != cudaSuccess || st != cudaStreamCaptureStatusNone;
}
inline long long capped_grid(long long grid, long long items) {
    if (g_items_cap > 0) {
        const long long g2 = (items + g_items_cap - 1) / g_items_cap;
        if (g2 > grid) grid = g2;
    }
    return grid;
}

inline int copy_stream(CopyStream **out, int which = 0, int prio_rank = -1) {   // which: pipeline lane
    static std::map<std::tuple<int, int, int>, CopyStream> m;
    int dev = 0;
    CK(cudaGetDevice(&dev));
    CopyStream &c = m[std::make_tuple(dev, which, prio_rank)];
    if (!c.s) {
        if (make_stream(&c.s, prio_rank)) return SNTRUP_E_CUDA;
        g_copy_streams.push_back(c.s);
        for (int i = 0; i < 2; i++) {
            CK(cudaEventCreateWithFlags(&c.comp[i], cudaEventDisableTiming));
            CK(cudaEventCreateWithFlags(&c.copy[i], cudaEventDisableTiming));
        }
    }
    *out = &c;
    return SNTRUP_OK;
}

// ------------------------------------------------------------------------------ aux stream
// Keygen's u_i = g_i * 3 f_{i^1} products depend only on the sample: they run on an aux stream
// concurrently with the (latency-bound) joint root inversion.  One per device.
struct AuxStream { cudaStream_t s = nullptr; cudaEvent_t go = nullptr, done = nullptr; };
inline int aux_stream(AuxStream **out) {
    static std::map<int, AuxStream> m;
    int dev = 0;
    CK(cudaGetDevice(&dev));
    AuxStream &x = m[dev];
    if (!x.s) {
        CK(cudaStreamCreateWithFlags(&x.s, cudaStreamNonBlocking));
        CK(cudaEventCreateWithFlags(&x.go, cudaEventDisableTiming));
        CK(cudaEventCreateWithFlags(&x.done, cudaEventDisableTiming));
    }
    *out = &x;
    return SNTRUP_OK;
}

// side stream on which asynchronous host-output calls record their completion event, and an
// event marking the end of the call's work on the caller's stream
inline int done_stream(cudaStream_t *out, cudaEvent_t *s0_end) {
    static std::map<int, std::pair<cudaStream_t, cudaEvent_t>> m;
    int dev = 0;
    CK(cudaGetDevice(&dev));
    auto &x = m[dev];
    if (!x.first) {
        CK(cudaStreamCreateWithFlags(&x.first, cudaStreamNonBlocking));
        CK(cudaEventCreateWithFlags(&x.second, cudaEventDisableTiming));
    }
    *out = x.first;
    *s0_end = x.second;
    return SNTRUP_OK;
}

// ------------------------------------------------------------------------------ workspace
// One cached workspace per (device, caller stream): calls on different streams never share
// scratch memory, so asynchronous calls on different streams are independent (the header's
// promise).  The workspace of the current call is selected by ws_reserve (under g_mu).
struct Workspace {
    char *base = nullptr;
    size_t cap = 0, used = 0;
    int dev = -1;
};
inline std::map<std::pair<int, uintptr_t>, Workspace> g_wsmap;
// bumped whenever a cached workspace is (re)allocated or released: captured keygen graphs
// (SNTRUP_OPT_GRAPH) hold workspace pointers and are rebuilt when it changes
inline uint64_t g_ws_epoch = 1;
inline Workspace *g_ws = nullptr;
inline Workspace g_user_ws;                          // a caller-supplied workspace (opts.workspace)

// bytes ws_reserve allocates for a request of `bytes` (slack so that slightly larger later
// calls on the same stream reuse the allocation)
inline size_t ws_alloc_bytes(size_t bytes) { return bytes + (bytes >> 3) + (1 << 20); }

inline int ws_reserve(size_t bytes, cudaStream_t stream, void *user = nullptr, size_t user_bytes = 0) {
    int dev;
    CK(cudaGetDevice(&dev));
    if (user) {                               // caller-owned memory: no caching, no allocation
        if (user_bytes < bytes) return SNTRUP_E_WORKSPACE;
        if ((uintptr_t)user & 255) return SNTRUP_E_ARG;
        g_user_ws.base = (char *)user;
        g_user_ws.cap = user_bytes;
        g_user_ws.used = 0;
        g_user_ws.dev = dev;
        g_ws = &g_user_ws;
        return SNTRUP_OK;
    }
    Workspace &w = g_wsmap[std::make_pair(dev, (uintptr_t)stream)];
    g_ws = &w;
    if (w.base && w.cap >= bytes) { w.used = 0; return SNTRUP_OK; }
    if (w.base) {
        CK(cudaDeviceSynchronize());          // in-flight work (any internal stream) may use it
        cudaFree(w.base);
        w.base = nullptr;
        w.cap = 0;
    }
    size_t cap = ws_alloc_bytes(bytes);
    ++g_ws_epoch;
    if (cudaMalloc(&w.base, cap) != cudaSuccess) {
        cudaGetLastError();
        w.base = nullptr;
        w.cap = 0;
        return SNTRUP_E_WORKSPACE;
    }
    w.cap = cap;
    w.used = 0;
    w.dev = dev;
    return SNTRUP_OK;
}

// Host-output staging (device buffers the D2H copies read from) lives in its own allocation per
// (device, caller stream), NOT in the workspace: asynchronous host-output calls leave their copies
// running after return, and the next call on the stream reuses the workspace at once.  Within a
// fixed layout each staging buffer is waited for (its copy-done event) right before its first
// write; a layout change (chunk, lanes, sizes) or growth first waits for every copy in flight.
struct Staging {
    char *base = nullptr;
    size_t cap = 0;
    uint64_t layout = 0;
};
inline std::map<std::pair<int, uintptr_t>, Staging> g_stmap;

inline int staging_reserve(size_t bytes, uint64_t layout, cudaStream_t stream, char **out) {
    int dev;
    CK(cudaGetDevice(&dev));
    Staging &st = g_stmap[std::make_pair(dev, (uintptr_t)stream)];
    if (st.base && st.cap >= bytes && st.layout == layout) { *out = st.base; return SNTRUP_OK; }
    for (cudaStream_t cs : g_copy_streams) CK(cudaStreamSynchronize(cs));   // copies still reading it
    if (st.base && st.cap < bytes) {
        cudaFree(st.base);
        st.base = nullptr;
        st.cap = 0;
    }
    if (!st.base) {
        if (cudaMalloc(&st.base, bytes) != cudaSuccess) {
            cudaGetLastError();
            st.base = nullptr;
            return SNTRUP_E_WORKSPACE;
        }
        st.cap = bytes;
    }
    st.layout = layout;
    *out = st.base;
    return SNTRUP_OK;
}

template <class T>
T *ws_take(size_t count) {
    size_t bytes = (count * sizeof(T) + 255) & ~(size_t)255;
    T *p = (T *)(g_ws->base + g_ws->used);
    g_ws->used += bytes;
    return p;
}

// every ws_take of a call stayed inside the reservation (checked before the first launch)
inline bool ws_fits() { return g_ws && g_ws->used <= g_ws->cap; }

inline size_t align256(size_t b) { return (b + 255) & ~(size_t)255; }

// ------------------------------------------------------------------------------ tree plan
// rows r.. of a row descriptor
inline RowDesc row_offset(RowDesc d, long long r) {
    if (d.ptr) d.ptr = (const uint8_t *)d.ptr + r * d.stride * d.bytes;
    return d;
}

struct TreePlan {
    int L;                          // levels = log2(B)
    std::vector<long long> cnt;     // cnt[0] = leaves, cnt[l] = ceil(cnt[l-1]/2)
    long long inner_rows() const { long long s = 0; for (int l = 1; l <= L; l++) s += cnt[l]; return s; }
};

inline TreePlan make_plan(long long m, int B) {
    TreePlan t;
    t.L = 0;
    while ((1 << t.L) < B) t.L++;
    t.cnt.resize(t.L + 1);
    t.cnt[0] = m;
    for (int l = 1; l <= t.L; l++) t.cnt[l] = (t.cnt[l - 1] + 1) / 2;
    return t;
}

// ------------------------------------------------------------------------------ launches
// ring-product implementation (sntrup_set_mul_impl): 0 = tensor cores, fp4 (tc4mul.cuh) where an
// operand is small + int8 (tcmul.cuh) otherwise, shared-A down-sweep; 1 = int32 schoolbook;
// 2 = int8 tensor cores only, one product per work item; 3 = int8 tensor cores with shared A;
// 4 = as 0 but big x small products also on fp4 (base-9 digits; slower, kept for A/B);
// 5 = as 0 but int8 products with MMA M = 64 (A/B for the M = 128 choice);
// 6 = as 0 but one int8 big x big product per work item (A/B for the shared-A down-sweep);
// 7 = as 0 but the keygen's u products fused with the R/q tree's level 1 (shared A; A/B);
// 8 = as 0 but the int8 big x big products software-pipelined (two operand stages, 8 warps)
inline int g_mul_impl = 0;
inline int g_divstep_threads = 256;
// root inversions when the roots are few (sntrup_set_root_impl): 0 = automatic (jump-divsteps,
// jump.cuh, for the standalone reciprocal calls and keygen calls of <= 4096 keys; one divstep at
// a time inside larger keygen calls), 1 = one
// divstep at a time everywhere (R/q: divstep_cta_kernel, one CTA barrier per step; R/3: the
// bitsliced warp divstep_kernel), 2 = jump-divsteps everywhere; + 4: the jump CTAs reserve only the
// shared memory they use (other kernels' CTAs may share their SMs) instead of more than half an SM
inline int g_root_impl = 0;
// per (device, caller stream): the device error flags of the last keygen call (asynchronous calls
// do not read them; sntrup_async_error does, once the call's work has completed)
inline std::map<std::pair<int, uintptr_t>, std::vector<int *>> g_async_err;                // R/q root CTA size (A/B knob; sntrup761 only)
inline unsigned long long *g_ws_trace = nullptr;   // SNTRUP_WS_TRACE: device [160][16] role cycles

struct DevInfo { int sms = 0; };
inline DevInfo &dev_info() {
    static std::map<int, DevInfo> m;
    int dev = 0;
    cudaGetDevice(&dev);
    DevInfo &d = m[dev];
    if (!d.sms) cudaDeviceGetAttribute(&d.sms, cudaDevAttrMultiProcessorCount, dev);
    return d;
}

// Resident 128-thread CTAs per SM of a persistent tensor-core kernel: the minimum of the
// shared-memory (1 KB reserved per CTA), register-file and TMEM-column (512 per SM) limits.  A
// persistent grid larger than what is resident runs a second partial wave after the first CTAs
// finish their whole share, so this must not over-count.
template <class F>
int resident_ctas(F kern, int smem, int tcols, int threads = 128) {
    cudaFuncAttributes fa;
    if (cudaFuncGetAttributes(&fa, kern) != cudaSuccess) return 1;
    const int regs = (fa.numRegs + 7) / 8 * 8;                  // allocation granularity
    const int by_regs = regs > 0 ? 65536 / (regs * threads) : 32;
    const int by_smem = (227 * 1024) / (smem + 1024);
    int nb = by_regs < by_smem ? by_regs : by_smem;
    if (nb * tcols > 512) nb = 512 / tcols;
    return nb < 1 ? 1 : nb;
}

template <class PS, int M, int LA, int LB, int NPR = 1, int MM = 128, bool XOPS = false, int NT = 128, int ST = 1,
          int NH = 1>
int launch_tc_impl(const MulArgs &a, cudaStream_t s) {
    using G = TcGeom<PS, LA, LB, NPR, MM>;
    constexpr int SMEM = tc_smem_bytes<G, LA, LB, NPR, ST, MM, NH>();
    auto kern = tc_mul_kernel<PS, M, LA, LB, NPR, MM, XOPS, NT, ST, NH>;
    static std::map<int, int> per_sm;                 // device -> resident CTAs per SM
    int dev = 0;
    CK(cudaGetDevice(&dev));
    auto it = per_sm.find(dev);
    if (it == per_sm.end()) {
        CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM));
        CK(cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout, 100));
        int nb = 0;
        nb = resident_ctas(kern, SMEM, tc_tmem_cols<G, LA, ST>(), NT);
        it = per_sm.emplace(dev, nb).first;
    }
    long long grid = capped_grid((long long)it->second * dev_info().sms, a.n_out);
    if (grid > a.n_out) grid = a.n_out;
    g_cur_kind = PK_I8;
    // per work item: NKS K steps x LA A-limbs, each MMA reading an MM x 32-byte A tile and an
    // NB x 32-byte B tile from shared memory
    g_cur_smem = (double)a.n_out * G::NKS * LA * (double)(MM * 32 + G::NB * 32);
    kern<<<(unsigned)grid, NT, SMEM, s>>>(a);
    LAUNCHED();
    return SNTRUP_OK;
}

// transposed form (tcxmul.cuh): one product per item, u = window operand (LA limbs), v = Z operand
template <class PS, int M, int LA, int LB, int NPR = 1, bool XOPS = false>
int launch_tcx_impl(const MulArgs &a, cudaStream_t s) {
    using G = TcxGeom<PS, LA, LB, NPR>;
    auto kern = tcx_mul_kernel<PS, M, LA, LB, NPR, XOPS>;
    static std::map<int, int> per_sm;
    int dev = 0;
    CK(cudaGetDevice(&dev));
    auto it = per_sm.find(dev);
    if (it == per_sm.end()) {
        CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, G::SMEM));
        CK(cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout, 100));
        it = per_sm.emplace(dev, resident_ctas(kern, G::SMEM, G::TCOLS)).first;
    }
    long long grid = capped_grid((long long)it->second * dev_info().sms, a.n_out);
    if (grid > a.n_out) grid = a.n_out;
    g_cur_kind = PK_I8;
    // per work item: NKS K steps x LB chains, each MMA reading an MM x 32-byte Z tile and an
    // NB x 32-byte window tile from shared memory
    g_cur_smem = (double)a.n_out * G::NKS * NPR * LB * (double)(G::MM * 32 + G::NB * 32);
    kern<<<(unsigned)grid, 128, G::SMEM, s>>>(a);
    LAUNCHED();
    return SNTRUP_OK;
}

// KEM-core pre/post-ops need the XOPS instantiation (keygen never sets them)
inline bool mul_xops(const MulArgs &a) { return a.round3 || a.X.mod3 || a.Y.mod3; }

// KEM pre/post-ops exist only in one-product-per-item M = 128 instantiations (the shapes the KEM
// core launches); an A/B variant asked to run them falls back to that kernel
template <class PS, int M, int LA, int LB, int NPR = 1>
int launch_tcx(const MulArgs &a, cudaStream_t s) {
    if (mul_xops(a)) return launch_tcx_impl<PS, M, LA, LB, 1, true>(a, s);
    return launch_tcx_impl<PS, M, LA, LB, NPR, false>(a, s);
}

template <class PS, int M, int LA, int LB, int NPR = 1, int MM = 128>
int launch_tc(const MulArgs &a, cudaStream_t s) {
    if (mul_xops(a)) return launch_tc_impl<PS, M, LA, LB, 1, 128, true>(a, s);
    return launch_tc_impl<PS, M, LA, LB, NPR, MM, false>(a, s);
}

// software-pipelined variant (two operand stages, 8 warps) of the int8 big x big products
template <class PS, int M, int NPR>
int launch_tc_pipe(const MulArgs &a, cudaStream_t s) {
    if (mul_xops(a)) return launch_tc_impl<PS, M, 2, 2, 1, 128, true>(a, s);
    return launch_tc_impl<PS, M, 2, 2, NPR, 128, false, 256, 2>(a, s);
}

template <class PS, int M, int LB, int NPR = 1, bool XOPS = false, int TA = 0, bool RING = false>
int launch_tc4_impl(const MulArgs &a, cudaStream_t s) {
    using G = Tc4Geom<PS, LB, NPR, TA>;
    auto kern = tc4_mul_kernel<PS, M, LB, NPR, XOPS, TA, RING>;
    static std::map<int, int> per_sm;
    int dev = 0;
    CK(cudaGetDevice(&dev));
    auto it = per_sm.find(dev);
    if (it == per_sm.end()) {
        CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, G::SMEM));
        CK(cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout, 100));
        int nb = 0;
        nb = resident_ctas(kern, G::SMEM, G::TCOLS);
        it = per_sm.emplace(dev, nb).first;
    }
    long long grid = capped_grid((long long)it->second * dev_info().sms, a.n_out);
    if (grid > a.n_out) grid = a.n_out;
    g_cur_kind = PK_F4;
    // per work item: NKS MMAs, each an 128 x 32-byte A tile (64 fp4 K-elements; none for the K
    // steps whose A is in TMEM) and an NB x 32-byte B tile
    g_cur_smem = (double)a.n_out * ((double)(RING ? 0 : G::NKS - G::NTA) * 128 * 32 + (double)G::NKS * G::NB * 32);
    kern<<<(unsigned)grid, 128, G::SMEM, s>>>(a);
    LAUNCHED();
    return SNTRUP_OK;
}

// warp-specialised fp4 products with the Hankel A operand in TMEM (tc4w.cuh): one persistent CTA
// of 13 warps per SM
template <class PS, int M, int NPR>
int launch_tc4w(const MulArgs &a, cudaStream_t s) {
    using W = Tc4wGeom<PS, NPR>;
    auto kern = tc4w_mul_kernel<PS, M, NPR>;
    static std::map<int, bool> init;
    int dev = 0;
    CK(cudaGetDevice(&dev));
    if (!init[dev]) {
        CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, W::SMEM));
        init[dev] = true;
    }
    long long grid = (long long)W::CTAS * dev_info().sms;            // CTAS resident per SM
    if (grid > a.n_out) grid = a.n_out;
    g_cur_kind = PK_F4;
    g_cur_smem = (double)a.n_out * (double)W::G::NKS * W::G::NB * 32;   // B tiles only: A is in TMEM
    MulArgs b = a;
    b.trace = g_ws_trace;
    kern<<<(unsigned)grid, W::THREADS, W::SMEM, s>>>(b);
    LAUNCHED();
    return SNTRUP_OK;
}

template <class PS, int M, int LB, int NPR = 1>
int launch_tc4(const MulArgs &a0, cudaStream_t s) {
    MulArgs a = a0;
    a.trace = g_ws_trace;                                 // phase timing in SNTRUP_WS_TRACE builds
    if (mul_xops(a)) return launch_tc4_impl<PS, M, LB, 1, true>(a, s);   // KEM: one product per item
    if constexpr (LB == 1) {
        // (int8 operand rows only: the kernel bulk-copies raw rows)
        if (g_mul_impl == 11 && a.mode != MUL_UP0 && a.X.bytes == 1 && (a.Y.bytes == 1 || a.mode == MUL_PAIRS))
            return launch_tc4w<PS, M, NPR>(a, s);
    }
    if constexpr (LB == 1 && PS::P == 761) {              // A/B variants: sntrup761 only
        if (g_mul_impl == 9) return launch_tc4_impl<PS, M, LB, NPR, false, 128>(a, s);  // A in TMEM, 128 cols
        if (g_mul_impl == 10) return launch_tc4_impl<PS, M, LB, NPR, false, 64>(a, s);  // A in TMEM, 64 cols
        if (g_mul_impl == 12) return launch_tc4_impl<PS, M, LB, NPR, false, 64, true>(a, s);  // all A via TMEM
    }
    return launch_tc4_impl<PS, M, LB, NPR, false>(a, s);
}

// The A/B-only ring-product variants (sntrup_set_mul_impl 2-10) are compiled for sntrup761 only;
// the other parameter sets run the default tensor-core path (or the int32 schoolbook, impl 1).
template <class PS>
constexpr bool kABVariants = PS::P == 761;

// la / lb: int8 limbs of the first / second operand (1 = small: R/3, 3f, g; 2 = R/q element).
template <class PS, int M>
int launch_mul(MulArgs a, cudaStream_t s, int la = 2, int lb = 2) {
    if (a.n_out <= 0) return SNTRUP_OK;
    if (g_route_on) {                        // tree tops on the chain's high-priority stream
        cudaStream_t t;
        if (int rc = route_stream(s, a.n_out <= g_top_items, &t)) return rc;
        s = t;
    }
    constexpr bool AB = kABVariants<PS>;
    const int sel = AB ? g_mul_impl : (g_mul_impl == 1 ? 1 : 0);
    const int impl = (sel >= 7) ? 0 : sel;   // 7-16: as 0 except u / pipelining / TMEM A / transposed
    const bool pipe = sel == 8;
    const bool tcx = sel == 13;              // one-product int8 items in the transposed form (tcxmul.cuh)
    // int8 big x big items with the K range in parts (default: two-product items in 2 parts):
    // 14 = one part (the former default), 15 = 3 parts, 16 = one-product items in 2 parts too
    // algorithmic ops: the method's work, 2 p^2 (p^2 multiply-adds) per ring product whatever the
    // implementation (limbs, digits, padding and the zero triangles are implementation overhead)
    ProfScope ps_(M == 3 ? PC_MUL_R3 : PC_MUL_RQ, (double)a.n_out, s, 2.0 * PS::P * PS::P * (double)a.n_out);
    if (impl == 1) {
        const int threads = (PS::P8 / 8 + 31) / 32 * 32;
        long long grid = a.n_out;
        if (grid > (1LL << 30)) grid = 1LL << 30;
        g_cur_kind = PK_I32;
        ring_mul_kernel<PS, M><<<(unsigned)grid, threads, 0, s>>>(a);
        LAUNCHED();
        return SNTRUP_OK;
    }
    // down-sweep with both operands of one kind: the two children of a parent share the parent's
    // inverse as the A operand (one work item per parent), halving the A-operand fetch that
    // bounds the tensor-core products.  int8 big x big at M = 128 too since the folded B operand
    // halved N (3 CTAs/SM); impl 6 keeps one big x big product per item for A/B.
    // (only where two such CTAs fit an SM; with the operands in two K parts that holds for every set,
    // p = 1277 included: 12.1 vs 10.95 M keys/s there, profiles/r02s3/kparts_1277.log)
    const bool big2 = la == 2 && lb == 2 && impl != 5 && impl != 6 &&
                      TcParts<TcGeom<PS, 2, 2, 2>, 2, 2, 2, 128, 2>::BY_SMEM >= 2;
    const bool down2 = (a.mode == MUL_DOWN || a.mode == MUL_DOWNH) && (M == 3 || (la == 1 && lb == 1) || big2) &&
                       impl != 2;
    if (down2) {
        a.mode = a.mode == MUL_DOWN ? MUL_DOWN2 : MUL_DOWNH2;
        a.n_out = (a.cnt_in + 1) / 2;
    }
    const bool fp4 = impl == 0 || impl == 4 || impl == 5 || impl == 6;
    if constexpr (M == 3) {
        a.swap = 0;
        if constexpr (AB) {
            if (!fp4) return down2 ? launch_tc<PS, M, 1, 1, 2>(a, s) : launch_tc<PS, M, 1, 1>(a, s);
        }
        return down2 ? launch_tc4<PS, M, 1, 2>(a, s) : launch_tc4<PS, M, 1, 1>(a, s);
    } else {
        constexpr int D9 = digits9(M);
        if (la == 1 && lb == 1) {
            a.swap = 0;
            if constexpr (AB) {
                if (!fp4) return down2 ? launch_tc<PS, M, 1, 1, 2>(a, s) : launch_tc<PS, M, 1, 1>(a, s);
            }
            return down2 ? launch_tc4<PS, M, 1, 2>(a, s) : launch_tc4<PS, M, 1, 1>(a, s);
        }
        if (la == 1 || lb == 1) {
            // the small operand takes the A (Hankel) role.  int8 with two limbs for the big one:
            // measured faster than fp4 with D9 base-9 digits (larger N, digit staging), see
            // DESIGN.md section 6; the fp4 variant stays selectable for A/B (impl 4); int8 products
            // at MMA M = 64 (half the A bytes per MMA, twice the N) are A/B mode impl 5
            a.swap = la == 1 ? 0 : 1;
            if constexpr (AB) {
                if (tcx) {                   // the big operand takes the window role (2 limbs along N)
                    a.swap = la == 1 ? 1 : 0;
                    return launch_tcx<PS, M, 2, 1>(a, s);
                }
                if (impl == 4) return launch_tc4<PS, M, D9, 1>(a, s);
                if (impl == 5) return launch_tc<PS, M, 1, 2, 1, 64>(a, s);
            }
            return launch_tc<PS, M, 1, 2>(a, s);
        }
        a.swap = 0;
        if constexpr (AB) {
            if (pipe) return down2 ? launch_tc_pipe<PS, M, 2>(a, s) : launch_tc_pipe<PS, M, 1>(a, s);
            if (impl == 5) return launch_tc<PS, M, 2, 2, 1, 64>(a, s);
        }
        if constexpr (AB) {
            if (tcx) return down2 ? launch_tcx<PS, M, 2, 2, 2>(a, s) : launch_tcx<PS, M, 2, 2>(a, s);
        }
        if constexpr (AB) {
            if (down2 && !mul_xops(a)) {
                if (sel == 14) return launch_tc_impl<PS, M, 2, 2, 2>(a, s);                                  // one part
                if (sel == 15) return launch_tc_impl<PS, M, 2, 2, 2, 128, false, 128, 1, 3>(a, s);
            }
            if (sel == 16 && !down2 && !mul_xops(a)) return launch_tc_impl<PS, M, 2, 2, 1, 128, false, 128, 1, 2>(a, s);
        }
        // two-product items: operands built and multiplied in two parts of the K range (half-size
        // buffers: 43 instead of 72 KB per CTA at p = 761, 5 resident CTAs per SM instead of 3)
        if (down2 && !mul_xops(a)) return launch_tc_impl<PS, M, 2, 2, 2, 128, false, 128, 1, 2>(a, s);
        if (down2) return launch_tc<PS, M, 2, 2, 2>(a, s);
        return launch_tc<PS, M, 2, 2>(a, s);
    }
}

template <class PS, int M>
int launch_divstep(const InvArgs &a, cudaStream_t s, bool bulk = false) {
    if (a.n <= 0) return SNTRUP_OK;
    if (g_route_on) {                        // roots: with the tree tops
        cudaStream_t t;
        if (int rc = route_stream(s, true, &t)) return rc;
        s = t;
    }
    // jump-divsteps when the roots are few and the call waits on them (the standalone reciprocal
    // calls, latency-sized keygen calls); inside a bulk keygen call the roots overlap the other
    // ring's products, where the per-step kernels' smaller SM footprint wins
    const int rmode = g_root_impl & 3;
    const bool jump = a.n < 2LL * dev_info().sms && (rmode == 2 || (rmode == 0 && !bulk));
    ProfScope ps_(M == 3 ? PC_INV_R3 : PC_INV_RQ, (double)a.n, s);
    if constexpr (M == 3) {
        if (jump) {
            CK((launch_jump_roots<PS, M>(a, s, !(g_root_impl & 4))));                                  // few roots: jump-divsteps
        } else {
            divstep_kernel<PS, M><<<(unsigned)((a.n + 3) / 4), 128, 0, s>>>(a);  // bitsliced, warp/root
        }
    } else {
        // few roots: latency bound -> one CTA of 8 warps per root; many roots: throughput bound
        // -> one warp per root (less per-step overhead in total)
        if (jump) {
            CK((launch_jump_roots<PS, M>(a, s, !(g_root_impl & 4))));
        } else if (a.n < 2LL * dev_info().sms)
        {
            // threads per root (A/B knob, sntrup_set_divstep_threads; default 256 = 8 warps)
            if constexpr (PS::P == 761) {
                if (g_divstep_threads == 128) { divstep_cta_kernel<PS, M, 128><<<(unsigned)a.n, 128, 0, s>>>(a); }
                else if (g_divstep_threads == 512) { divstep_cta_kernel<PS, M, 512><<<(unsigned)a.n, 512, 0, s>>>(a); }
                else if (g_divstep_threads == 768) { divstep_cta_kernel<PS, M, 768><<<(unsigned)a.n, 768, 0, s>>>(a); }
                else divstep_cta_kernel<PS, M, 256><<<(unsigned)a.n, 256, 0, s>>>(a);
            } else {
                divstep_cta_kernel<PS, M, 256><<<(unsigned)a.n, 256, 0, s>>>(a);
            }
        }
        else
            divstep_kernel<PS, M><<<(unsigned)((a.n + 3) / 4), 128, 0, s>>>(a);
    }
    LAUNCHED();
    return SNTRUP_OK;
}

inline RowDesc rows8(const void *p, long long stride, int scale = 1) { return RowDesc{p, stride, 1, scale}; }
inline RowDesc rows16(const void *p, long long stride) { return RowDesc{p, stride, 2, 1}; }

// Batch inversion over one ring by product trees.  X0 = leaves (row descriptor), out0 = leaf
// inverse rows.  Levels l >= 1 live in lvl[l] / inv[l].  M = ring modulus (3 or q).  Split into
// up-sweep / roots / down-sweep so that keygen can invert both rings' roots in one launch.
template <class PS, int M>
struct TreeJob {
    const TreePlan &tp;
    RowDesc X0;
    void *out0;
    int out_bytes;
    long long out_stride;
    const std::vector<void *> &lvl, &inv;
    uint8_t *root_ok;
    bool leaves_small;

    long long stride() const { return out_bytes == 2 ? PS::P8 : PS::P16; }
    RowDesc desc(int l) const {
        if (l == 0) return X0;
        return out_bytes == 2 ? rows16(lvl[l], stride()) : rows8(lvl[l], stride());
    }
    RowDesc idesc(int l) const {
        if (l == 0) return out_bytes == 2 ? rows16(out0, out_stride) : rows8(out0, out_stride);
        return out_bytes == 2 ? rows16(inv[l], stride()) : rows8(inv[l], stride());
    }
    int up(cudaStream_t s, uint64_t *nprod, int start = 1) const {
        int rc;
        for (int l = start; l <= tp.L; l++) {
            MulArgs a{};
            a.mode = MUL_PAIRS;
            a.n_out = tp.cnt[l];
            a.cnt_in = tp.cnt[l - 1];
            a.X = desc(l - 1);
            a.out = lvl[l];
            a.out_stride = stride();
            a.out_bytes = out_bytes;
            a.periodic = (M != 3) && !(l == 1 && leaves_small);
            const int lx = (M == 3 || (l == 1 && leaves_small)) ? 1 : 2;
            if ((rc = launch_mul<PS, M>(a, s, lx, lx))) return rc;
            *nprod += tp.cnt[l - 1] / 2;
        }
        return SNTRUP_OK;
    }
    InvArgs roots() const {
        const int L = tp.L;
        InvArgs ia{};
        ia.n = tp.cnt[L];
        ia.in = desc(L);
        ia.out = L == 0 ? out0 : inv[L];
        ia.out_stride = L == 0 ? out_stride : stride();
        ia.out_bytes = out_bytes;
        ia.ok = root_ok;
        return ia;
    }
    int down(cudaStream_t s, uint64_t *nprod, int stop = 1) const {
        return down_group(s, nprod, tp.L, stop, 0, tp.cnt[tp.L]);
    }
    // Levels hi .. lo of the down-sweep restricted to the subtrees of roots [ra, rb): at level l
    // they own rows [ra << (L-l), rb << (L-l)) (a contiguous range of every level).
    int down_group(cudaStream_t s, uint64_t *nprod, int hi, int lo, long long ra, long long rb) const {
        int rc;
        for (int l = hi; l >= lo; l--) {
            const long long r0 = ra << (tp.L - l + 1);
            long long r1 = rb << (tp.L - l + 1);
            if (r1 > tp.cnt[l - 1]) r1 = tp.cnt[l - 1];
            if (r1 <= r0) continue;
            MulArgs a{};
            a.mode = MUL_DOWN;
            a.n_out = r1 - r0;
            a.cnt_in = r1 - r0;
            a.X = row_offset(desc(l - 1), r0);
            a.Y = row_offset(idesc(l), r0 / 2);
            const RowDesc od = row_offset(idesc(l - 1), r0);
            a.out = const_cast<void *>(od.ptr);
            a.out_stride = od.stride;
            a.out_bytes = out_bytes;
            a.periodic = (M != 3) && !(l == 1 && leaves_small);
            // operands: (inverse of the parent: big) x (sibling: small at level 1 over small leaves)
            const int lsib = (M == 3 || (l == 1 && leaves_small)) ? 1 : 2;
            if ((rc = launch_mul<PS, M>(a, s, M == 3 ? 1 : 2, lsib))) return rc;
            *nprod += ((r1 - r0) / 2) * 2;
        }
        return SNTRUP_OK;
    }
};

template <class PS, int M>
int batch_inverse(const TreePlan &tp, RowDesc X0, void *out0, int out_bytes, long long out_stride,
                  const std::vector<void *> &lvl, const std::vector<void *> &inv, uint8_t *root_ok,
                  bool leaves_small, cudaStream_t s, uint64_t *nprod) {
    const TreeJob<PS, M> j{tp, X0, out0, out_bytes, out_stride, lvl, inv, root_ok, leaves_small};
    int rc;
    if ((rc = j.up(s, nprod))) return rc;
    if ((rc = launch_divstep<PS, M>(j.roots(), s))) return rc;
    return j.down(s, nprod);
}

// Both rings' roots in one launch (keygen).
// (256 threads per block measured best against 128 and 512: profiles/)
template <class PS>
int launch_joint_roots(const InvArgs &r3, const InvArgs &rq, cudaStream_t s) {
    constexpr int NT = 256, WPB = NT / 32;
    const int nb3 = (int)((r3.n + WPB - 1) / WPB);
    const int rq_cta = rq.n < 2LL * dev_info().sms ? 1 : 0;
    const long long nbq = rq_cta ? rq.n : (rq.n + WPB - 1) / WPB;
    ProfScope ps_(PC_INV_R3, (double)(r3.n + rq.n), s);
    joint_roots_kernel<PS, NT><<<(unsigned)(nb3 + nbq), NT, 0, s>>>(r3, rq, nb3, rq_cta);
    LAUNCHED();
    return SNTRUP_OK;
}

// ------------------------------------------------------------------------------ keygen
// Per pipeline lane: a stream, an aux stream (u products) and one chunk's workspace.  With two
// or more chunks, consecutive chunks alternate between two lanes (the caller's stream and an
// internal stream), so one chunk's latency-bound phases (sampling, tree tops, root inversion)
// overlap the other chunk's tensor-core products.
struct Lane {
    cudaStream_t s = nullptr;
    AuxStream *ax = nullptr;
    AuxStream *r3 = nullptr;       // SNTRUP_OPT_RING_STREAMS: the R/3 chain's stream + events
    int8_t *G = nullptr, *F = nullptr, *Ginv = nullptr;
    uint8_t *att = nullptr;
    std::vector<void *> l3, i3, lq, iq;
    int16_t *Fbar = nullptr, *H = nullptr, *U = nullptr;
    uint8_t *ok3 = nullptr, *okq = nullptr;
    unsigned long long *repaired = nullptr;
    int *err = nullptr;
};

// internal lane li: a stream and its own aux stream (per device, per priority mode)
inline int lane_streams(int li, int prio_rank, cudaStream_t *s2, AuxStream **ax2) {
    static std::map<std::tuple<int, int, int>, std::pair<cudaStream_t, AuxStream>> m;
    int dev = 0;
    CK(cudaGetDevice(&dev));
    auto &e = m[std::make_tuple(dev, li, prio_rank)];
    if (!e.first) {
        if (make_stream(&e.first, prio_rank) || make_stream(&e.second.s, prio_rank)) return SNTRUP_E_CUDA;
        CK(cudaEventCreateWithFlags(&e.second.go, cudaEventDisableTiming));
        CK(cudaEventCreateWithFlags(&e.second.done, cudaEventDisableTiming));
    }
    *s2 = e.first;
    *ax2 = &e.second;
    return SNTRUP_OK;
}

// R/3-chain stream of a lane (SNTRUP_OPT_RING_STREAMS); go = sample done, done = R/3 chain done
inline int ring_stream(int lane, int prio_rank, AuxStream **out) {
    static std::map<std::tuple<int, int, int>, AuxStream> m;
    int dev = 0;
    CK(cudaGetDevice(&dev));
    AuxStream &x = m[std::make_tuple(dev, lane, prio_rank)];
    if (!x.s) {
        if (make_stream(&x.s, prio_rank)) return SNTRUP_E_CUDA;
        CK(cudaEventCreateWithFlags(&x.go, cudaEventDisableTiming));
        CK(cudaEventCreateWithFlags(&x.done, cudaEventDisableTiming));
    }
    *out = &x;
    return SNTRUP_OK;
}

constexpr int MAX_LANES = 4;
struct LaneJoin { cudaEvent_t start = nullptr, end[MAX_LANES] = {}, upd[MAX_LANES] = {}; };
inline int lane_join_events(LaneJoin **out) {
    static std::map<int, LaneJoin> m;
    int dev = 0;
    CK(cudaGetDevice(&dev));
    LaneJoin &j = m[dev];
    if (!j.start) {
        CK(cudaEventCreateWithFlags(&j.start, cudaEventDisableTiming));
        for (int i = 0; i < MAX_LANES; i++) {
            CK(cudaEventCreateWithFlags(&j.end[i], cudaEventDisableTiming));
            CK(cudaEventCreateWithFlags(&j.upd[i], cudaEventDisableTiming));
        }
    }
    *out = &j;
    return SNTRUP_OK;
}

// Shape of a keygen call: chunking, lanes, and the exact device bytes it reserves -- one helper
// for keygen_impl and sntrup_keygen_workspace_bytes, so the query is what a call takes.
struct KeygenShape {
    uint64_t chunk;
    size_t pkb, skb;
    int nl, nbuf;
    size_t ws_need;      // workspace (cached per stream, or the caller's)
    size_t stage_need;   // host-output staging (own allocation; 0 without SNTRUP_OPT_HOST_OUTPUT)
};

template <class PS>
KeygenShape keygen_shape(uint64_t n, int B, uint32_t flags, uint64_t chunk_keys, size_t pk_bytes) {
    KeygenShape k{};
    uint64_t chunk = chunk_keys ? chunk_keys : 65536;
    chunk = (chunk + B - 1) / B * B;
    if (chunk > n) chunk = (n + B - 1) / B * B;
    k.chunk = chunk;
    k.pkb = pk_bytes;
    k.skb = 2 * PS::SKH;
    const uint64_t nchunks = (n + chunk - 1) / chunk;
    const int nlmax = (flags & SNTRUP_OPT_SERIAL) ? 1 : (flags & SNTRUP_OPT_LANES4) ? 4 : 2;
    k.nl = (int)(nchunks < (uint64_t)nlmax ? nchunks : nlmax);
    k.nbuf = k.nl >= 2 ? k.nl : 2;          // host-output staging buffers (lane-owned if nl >= 2)
    // per lane, exactly the ws_take calls of keygen_impl (each rounded up to 256 bytes)
    const TreePlan tp = make_plan((long long)chunk, B);
    size_t per_lane = 3 * align256(chunk * PS::P16) + align256(chunk);           // G, F, Ginv, attempts
    for (int l = 1; l <= tp.L; l++)
        per_lane += 2 * align256(tp.cnt[l] * PS::P16) + 2 * align256(tp.cnt[l] * PS::P8 * 2);
    per_lane += 3 * align256(chunk * PS::P8 * 2);                                // Fbar, H, U
    per_lane += 2 * align256(tp.cnt[tp.L]);                                      // root ok flags
    per_lane += align256(sizeof(unsigned long long)) + align256(sizeof(int));    // counters
    k.ws_need = (size_t)k.nl * per_lane;
    k.stage_need = (flags & SNTRUP_OPT_HOST_OUTPUT)
                       ? (size_t)k.nbuf * (align256(chunk * k.pkb) + align256(chunk * k.skb)) : 0;
    // graph replay with host outputs: two whole-call device output sets (keygen_graph_host)
    if ((flags & SNTRUP_OPT_HOST_OUTPUT) && (flags & SNTRUP_OPT_GRAPH))
        k.stage_need = 2 * (align256(n * k.pkb) + align256(n * k.skb));
    return k;
}

template <class PS>
int keygen_impl(uint64_t n, uint64_t seed, uint8_t *pk_out, uint8_t *sk_out,
                const sntrup_keygen_opts &o) {
    int dev;
    CK(cudaGetDevice(&dev));
    DevTables *tb;
    int rc = build_tables(dev, PS::P, PS::WT, &tb);
    if (rc) return rc;
    const cudaStream_t s0 = (cudaStream_t)o.stream;
    const int B = o.batch_size ? (int)o.batch_size : 32;
    if (B < 1 || B > 4096 || (B & (B - 1))) return SNTRUP_E_ARG;
    const bool host_out = (o.flags & SNTRUP_OPT_HOST_OUTPUT) != 0;
    const KeygenShape ks = keygen_shape<PS>(n, B, o.flags, o.chunk_keys, tb->enc.pk_bytes);
    const uint64_t chunk = ks.chunk;
    const size_t pkb = ks.pkb, skb = ks.skb;
    const int nl = ks.nl, nbuf = ks.nbuf;
    const TreePlan tpmax = make_plan((long long)chunk, B);
    if ((rc = ws_reserve(ks.ws_need, s0, o.workspace, o.workspace_bytes))) return rc;
    char *stage_base = nullptr;
    if (host_out) {
        const uint64_t layout = ((uint64_t)PS::P << 48) ^ (chunk << 8) ^ (uint64_t)(nbuf << 4) ^ (uint64_t)nl;
        if ((rc = staging_reserve(ks.stage_need, layout, s0, &stage_base))) return rc;
    }
    Lane lanes[MAX_LANES];
    // tree tops and roots on high-priority companion streams (sntrup_set_sched): bulk calls with
    // ring streams only; not under graph capture or the serialised measurement pass
    struct RouteGuard {
        RouteGuard(bool on) { g_route_on = on; }
        ~RouteGuard() { g_route_on = false; }
    } route_guard(g_top_items > 0 && n > 4096 && (o.flags & SNTRUP_OPT_RING_STREAMS) &&
                  !(o.flags & SNTRUP_OPT_SERIAL) && !stream_capturing(s0));
    const bool prio = (o.flags & SNTRUP_OPT_LANE_PRIORITY) != 0;
    const int l0 = prio ? 0 : 1;           // first lane on an internal stream (forked from s0)
    for (int li = 0; li < nl; li++) {
        Lane &L = lanes[li];
        const int pr = prio ? (nl > 1 ? li * 8 / (nl - 1) : 0) : -1;
        if (li < l0) {
            L.s = s0;
            if ((rc = aux_stream(&L.ax))) return rc;
        } else {
            if ((rc = lane_streams(li, pr, &L.s, &L.ax))) return rc;
        }
        L.G = ws_take<int8_t>(chunk * PS::P16);
        L.F = ws_take<int8_t>(chunk * PS::P16);
        L.Ginv = ws_take<int8_t>(chunk * PS::P16);
        L.att = ws_take<uint8_t>(chunk);
        L.l3.assign(tpmax.L + 1, nullptr); L.i3.assign(tpmax.L + 1, nullptr);
        L.lq.assign(tpmax.L + 1, nullptr); L.iq.assign(tpmax.L + 1, nullptr);
        for (int l = 1; l <= tpmax.L; l++) {
            L.l3[l] = ws_take<int8_t>(tpmax.cnt[l] * PS::P16);
            L.i3[l] = ws_take<int8_t>(tpmax.cnt[l] * PS::P16);
            L.lq[l] = ws_take<int16_t>(tpmax.cnt[l] * PS::P8);
            L.iq[l] = ws_take<int16_t>(tpmax.cnt[l] * PS::P8);
        }
        L.Fbar = ws_take<int16_t>(chunk * PS::P8);
        L.H = ws_take<int16_t>(chunk * PS::P8);
        L.U = ws_take<int16_t>(chunk * PS::P8);
        L.ok3 = ws_take<uint8_t>(tpmax.cnt[tpmax.L]);
        L.okq = ws_take<uint8_t>(tpmax.cnt[tpmax.L]);
        L.repaired = ws_take<unsigned long long>(1);
        L.err = ws_take<int>(1);
        if ((o.flags & SNTRUP_OPT_RING_STREAMS) && !(o.flags & SNTRUP_OPT_SERIAL))
            if ((rc = ring_stream(li, pr, &L.r3))) return rc;
    }
    if (!ws_fits()) return SNTRUP_E_INTERNAL;    // keygen_shape and the takes above disagree
    uint8_t *pk_stage[MAX_LANES] = {}, *sk_stage[MAX_LANES] = {};
    CopyStream *csl[MAX_LANES] = {};               // one copy stream per lane: copies follow readiness
    if (host_out) {
        for (int i = 0; i < nbuf; i++) {
            pk_stage[i] = (uint8_t *)stage_base + i * (align256(chunk * pkb) + align256(chunk * skb));
            sk_stage[i] = pk_stage[i] + align256(chunk * pkb);
        }
        for (int li = 0; li < nl; li++)
            if ((rc = copy_stream(&csl[li], li, prio ? li : -1))) return rc;
        if (nl == 1) csl[1] = csl[0];
    }
    LaneJoin *lj = nullptr;
    if (nl > l0) {                         // internal lanes start after everything enqueued before the call
        if ((rc = lane_join_events(&lj))) return rc;
        CK(cudaEventRecord(lj->start, s0));
        for (int li = l0; li < nl; li++) CK(cudaStreamWaitEvent(lanes[li].s, lj->start, 0));
    }
    for (int li = 0; li < nl; li++) {
        CK(cudaMemsetAsync(lanes[li].repaired, 0, sizeof(unsigned long long), lanes[li].s));
        CK(cudaMemsetAsync(lanes[li].err, 0, sizeof(int), lanes[li].s));
    }

    uint64_t n_rq = 0, n_r3 = 0, n_inv = 0;
    for (uint64_t c0 = 0; c0 < n; c0 += chunk) {
        const uint64_t m = (n - c0 < chunk) ? n - c0 : chunk;
        const uint64_t first = o.first_key_index + c0;
        const TreePlan tp = make_plan((long long)m, B);
        const uint64_t ci = c0 / chunk;
        Lane &L = lanes[ci % nl];
        const cudaStream_t s = L.s;                          // this chunk's stream
        // host outputs: staging buffer ci mod nbuf (= the lane's own with >= 2 lanes, alternating
        // with one lane), reused nbuf chunks later after its copies; events by buffer parity
        const int sb = (int)(ci % nbuf), buf = sb & 1;
        int8_t *Gc = o.g_out ? o.g_out + c0 * PS::P16 : L.G;
        int8_t *Fc = o.f_out ? o.f_out + c0 * PS::P16 : L.F;
        int8_t *Ic = o.ginv_out ? o.ginv_out + c0 * PS::P16 : L.Ginv;
        uint8_t *Ac = o.attempts_out ? o.attempts_out + c0 : L.att;
        int16_t *Hc = o.h_out ? o.h_out + c0 * PS::P8 : L.H;
        CopyStream *cs = csl[ci % nl];
        // (host outputs: the staging buffer is free once its previous copies -- this call's, or an
        // earlier asynchronous call's -- are done; waited for right before its first write, so
        // the chunk's compute overlaps those copies)
        uint8_t *pkc = host_out ? pk_stage[sb] : pk_out + c0 * pkb;
        uint8_t *skc = host_out ? sk_stage[sb] : sk_out + c0 * skb;

        // SNTRUP_OPT_STAGGER: lane ci of the first round starts when lane ci-1 has finished its
        // R/q up-sweep, i.e. its sampling and up-sweeps fill the SMs lane ci-1's root inversion
        // leaves idle, and lane ci-1 (and its output) completes earlier
        const bool stagger = (o.flags & SNTRUP_OPT_STAGGER) && nl > 1;
        if (stagger && ci >= 1 && ci < (uint64_t)nl) CK(cudaStreamWaitEvent(s, lj->upd[ci - 1], 0));
        SampleArgs sa{};
        sa.seed = seed; sa.first = first; sa.n = m;
        sa.G = Gc; sa.F = Fc; sa.attempts = Ac;
        sa.T = tb->T; sa.masks = tb->masks; sa.nf = tb->nf;
        // The sampler's small-factor test only saves re-draws: the tree-root test + repair decide
        // invertibility exactly anyway.  Where a tree almost never fails
        // without it (761: 3^-19 per draw, 857: 3^-25), it is skipped.
        if (o.flags & SNTRUP_OPT_NO_SMALL_CHECK) sa.small_check = 0;
        else if (o.flags & SNTRUP_OPT_FORCE_SMALL_CHECK) sa.small_check = 1;
        else sa.small_check = (tb->p_small_reject * B > 1e-4) ? 1 : 0;
        sa.err = L.err;
        {
            ProfScope ps_(PC_SAMPLE, (double)m, s);
            sample_kernel<PS><<<(unsigned)((m + 3) / 4), 128, 0, s>>>(sa);
        }
        LAUNCHED();

        // R/3: Gbar = batchInv(G) (Algorithm 1 line 10); R/q: Fbar = batchInv([3 f]) (line 11).
        // Both trees up, both rings' roots in one launch, then the down-sweeps.
        //
        // h = g * fbar (line 12) is computed without fbar: at the bottom of the R/q tree
        // fbar_i = 1/(3 f_i) = P_j * 3 f_{i^1} with P_j the inverse of the leaves' parent, so
        // h_i = P_j * u_i with u_i = g_i * 3 f_{i^1}.  The u products (small x small, fp4) need only
        // the sample and run on an aux stream beside the root inversion; the bottom R/q down-sweep
        // level (1 x 2 limbs per product) disappears, h becomes a 2 x 2-limb product.
        // (B = 1 has no parents: plain fbar, then h = g * fbar.)
        const TreeJob<PS, 3> j3{tp, rows8(Gc, PS::P16), Ic, 1, PS::P16, L.l3, L.i3, L.ok3, true};
        const TreeJob<PS, PS::Q> jq{tp, rows8(Fc, PS::P16, 3), L.Fbar, 2, PS::P8, L.lq, L.iq, L.okq, true};
        const bool utrick = tp.L >= 1;
        const bool rings = L.r3 != nullptr;      // R/3 chain on its own stream
        const bool serial = (o.flags & SNTRUP_OPT_SERIAL) != 0;
        AuxStream *ax = L.ax;
        const cudaStream_t s3 = rings ? L.r3->s : s;  // stream of the R/3 chain
        if (rings) {
            CK(cudaEventRecord(L.r3->go, s));
            CK(cudaStreamWaitEvent(s3, L.r3->go, 0));
        }
        if ((rc = j3.up(s3, &n_r3))) return rc;
        // fp4 small x small paths: u_{2j} = g_{2j} * 3f_{2j+1} and the R/q tree's level 1,
        // 3f_{2j} * 3f_{2j+1}, share their A operand 3f_{2j+1} (one NPR = 2 work item), then the
        // odd u_{2j+1} = g_{2j+1} * 3f_{2j}: 2 A-operand fetches per leaf pair instead of 3
        // (A/B variant, impl 7: fewer A-operand fetches, but it moves the u products from the aux
        // stream -- where they fill the SMs the latency-bound root inversion leaves idle -- onto
        // the R/q chain's critical path; measured 2.5% slower than the default)
        const bool fused_u = utrick && g_mul_impl == 7 && kABVariants<PS>;
        if (fused_u) {
            MulArgs a{};
            a.mode = MUL_UP0;
            a.n_out = (long long)((m + 1) / 2);
            a.cnt_in = (long long)m;
            a.X = rows8(Gc, PS::P16);
            a.Y = rows8(Fc, PS::P16, 3);
            a.out = L.U;
            a.out_stride = PS::P8;
            a.out_bytes = 2;
            a.out2 = L.lq[1];
            a.out2_stride = PS::P8;
            {
                ProfScope ps_(PC_MUL_RQ, (double)(m + m / 2), s, 2.0 * PS::P * PS::P * (double)(m + m / 2));
                if ((rc = launch_tc4<PS, PS::Q, 1, 2>(a, s))) return rc;
            }
            if (m >= 2) {
                MulArgs b = a;
                b.mode = MUL_ODDSIB;
                b.n_out = (long long)(m / 2);
                b.out2 = nullptr;
                ProfScope ps_(PC_MUL_RQ, (double)(m / 2), s, 2.0 * PS::P * PS::P * (double)(m / 2));
                if ((rc = launch_tc4<PS, PS::Q, 1, 1>(b, s))) return rc;
            }
            CK(cudaEventRecord(ax->done, s));                   // u final (repair waits on it)
            n_rq += m / 2;                                       // level 1 (the u are counted below)
        }
        if ((rc = jq.up(s, &n_rq, fused_u ? 2 : 1))) return rc;
        if (stagger && ci + 1 < (uint64_t)nl) CK(cudaEventRecord(lj->upd[ci], s));
        if (utrick && !fused_u && serial) {
            // SNTRUP_OPT_SERIAL (measurement): the u products on the chunk's own stream, so every
            // kernel of the call runs alone and its CUDA-event time is its own
            MulArgs a{};
            a.mode = MUL_SIB;
            a.n_out = (long long)m;
            a.cnt_in = (long long)m;
            a.X = rows8(Gc, PS::P16);
            a.Y = rows8(Fc, PS::P16, 3);
            a.out = L.U;
            a.out_stride = PS::P8;
            a.out_bytes = 2;
            a.periodic = 0;
            if ((rc = launch_mul<PS, PS::Q>(a, s, 1, 1))) return rc;
            CK(cudaEventRecord(ax->done, s));
        } else if (utrick && !fused_u) {
            CK(cudaEventRecord(ax->go, s));
            CK(cudaStreamWaitEvent(ax->s, ax->go, 0));
            MulArgs a{};
            a.mode = MUL_SIB;
            a.n_out = (long long)m;
            a.cnt_in = (long long)m;
            a.X = rows8(Gc, PS::P16);
            a.Y = rows8(Fc, PS::P16, 3);
            a.out = L.U;
            a.out_stride = PS::P8;
            a.out_bytes = 2;
            a.periodic = 0;
            if ((rc = launch_mul<PS, PS::Q>(a, ax->s, 1, 1))) return rc;
            CK(cudaEventRecord(ax->done, ax->s));
        }
        if (rings || serial) {
            // each ring's roots on its own chain: one ring's latency-bound inversion overlaps the
            // other ring's products (serial: one after the other, separately timed)
            // a latency-sized call (<= 4096 keys) waits on its roots: jump-divsteps (automatic policy)
            const bool bulk = n > 4096;
            if ((rc = launch_divstep<PS, 3>(j3.roots(), s3, bulk))) return rc;
            if ((rc = launch_divstep<PS, PS::Q>(jq.roots(), s, bulk))) return rc;
        } else {
            if ((rc = launch_joint_roots<PS>(j3.roots(), jq.roots(), s))) return rc;
        }
        if ((rc = j3.down(s3, &n_r3))) return rc;
        if ((rc = route_flush(s3))) return rc;
        if (utrick) CK(cudaStreamWaitEvent(s3, ax->done, 0));    // repair may rewrite u rows
        RepairArgs ra{};
        ra.seed = seed; ra.first = first; ra.n = m; ra.B = B; ra.root_ok = L.ok3;
        ra.G = Gc; ra.Ginv = Ic; ra.attempts = Ac;
        ra.T = tb->T; ra.masks = tb->masks; ra.nf = tb->nf; ra.small_check = sa.small_check;
        ra.repaired = L.repaired; ra.err = L.err;
        ra.F = Fc; ra.U = utrick ? L.U : nullptr;
        {
            ProfScope ps_(PC_REPAIR, (double)m, s3);
            repair_kernel<PS><<<(unsigned)((m + 3) / 4), 128, 0, s3>>>(ra);
        }
        LAUNCHED();

        if (host_out) {
            // sk = Small(f) || Small(1/g) is final here (after repair): encode it and start its
            // D2H copy while the R/q tree runs
            CK(cudaStreamWaitEvent(s3, cs->copy[buf], 0));          // staging free
            EncArgs ea{};
            ea.n = m; ea.h = nullptr; ea.f = Fc; ea.ginv = Ic; ea.pk = nullptr; ea.sk = skc; ea.t = tb->enc;
            {
                ProfScope ps_(PC_ENCODE, (double)m, s3);
                encode_kernel<PS><<<(unsigned)((m + 3) / 4), 128, 0, s3>>>(ea);
            }
            LAUNCHED();
            CK(cudaEventRecord(cs->comp[buf], s3));
            CK(cudaStreamWaitEvent(cs->s, cs->comp[buf], 0));
            CK(cudaMemcpyAsync(sk_out + c0 * skb, skc, m * skb, cudaMemcpyDeviceToHost, cs->s));
        }
        // The R/q chain joins the R/3 chain (G, 1/g and u final after repair) only before its first
        // h product: the R/q down-sweep needs nothing from R/3, so it overlaps the R/3 down-sweep,
        // repair and sk encode.
        bool joined = !rings, pk_staging_free = false;
        if (rings) CK(cudaEventRecord(L.r3->done, s3));
        // H and encode (KeyGen step 5).  With host outputs the tail runs in groups of subtrees:
        // the bottom down-sweep levels (<= SG), h and the pk encode of group j complete before
        // group j+1 starts, so group j's pk slice is copied D2H while the next groups compute
        // (pk is 3/4 of the output bytes and only exists at the very end of its subtrees).
        // (asynchronous host-output calls overlap their copies with the next call instead)
        const bool async_req = host_out && (o.flags & SNTRUP_OPT_ASYNC) && o.done_event && !o.stats_out;
        const int nsub = (host_out && !async_req) ? 4 : 1;
        const long long nroots = tp.cnt[tp.L];
        const bool grouped = host_out && utrick && nroots >= nsub;
        const int SG = tp.L < 5 ? tp.L : 5;
        if ((rc = jq.down(s, &n_rq, grouped ? SG + 1 : (utrick ? 2 : 1)))) return rc;
        if ((rc = route_flush(s))) return rc;
        if (utrick) n_rq += m;                                     // the u products replace level 1
        n_inv += 2 * tp.cnt[tp.L];
        for (int j = 0; j < nsub; j++) {
            uint64_t r0, r1;
            if (grouped) {
                const long long ra = nroots * j / nsub, rb = nroots * (j + 1) / nsub;
                if ((rc = jq.down_group(s, &n_rq, SG, 2, ra, rb))) return rc;
                if ((rc = route_flush(s))) return rc;
                r0 = (uint64_t)ra << tp.L;
                r1 = (uint64_t)rb << tp.L;
                if (r1 > m) r1 = m;
            } else {
                r0 = (m * (uint64_t)j / nsub) & ~1ull;
                r1 = (j + 1 == nsub) ? m : ((m * (uint64_t)(j + 1) / nsub) & ~1ull);
            }
            const uint64_t rows = r1 > r0 ? r1 - r0 : 0;
            if (!rows) continue;
            if (!joined) {
                CK(cudaStreamWaitEvent(s, L.r3->done, 0));   // (also orders the sk staging write)
                joined = true;
            }
            if (host_out && !pk_staging_free) {
                CK(cudaStreamWaitEvent(s, cs->copy[buf], 0));   // pk staging free
                pk_staging_free = true;
            }
            {
                MulArgs a{};
                if (utrick) {
                    // h_i = P_{i/2} * u_i
                    const RowDesc P1 = jq.idesc(1);
                    a.mode = MUL_DOWNH;
                    a.n_out = (long long)rows;
                    a.cnt_in = (long long)rows;
                    a.X = rows16(L.U + r0 * PS::P8, PS::P8);
                    a.Y = rows16((const int16_t *)P1.ptr + (r0 / 2) * P1.stride, P1.stride);
                    a.periodic = 1;
                    a.out = Hc + r0 * PS::P8;
                    a.out_stride = PS::P8;
                    a.out_bytes = 2;
                    if ((rc = launch_mul<PS, PS::Q>(a, s, 2, 2))) return rc;
                } else {
                    a.mode = MUL_ZIP;
                    a.n_out = (long long)rows;
                    a.X = rows8(Gc + r0 * PS::P16, PS::P16);
                    a.Y = rows16(L.Fbar + r0 * PS::P8, PS::P8);
                    a.periodic = 0;
                    a.out = Hc + r0 * PS::P8;
                    a.out_stride = PS::P8;
                    a.out_bytes = 2;
                    if ((rc = launch_mul<PS, PS::Q>(a, s, 1, 2))) return rc;   // g small, fbar big
                }
            }
            if ((rc = route_flush(s))) return rc;
            {
                EncArgs ea{};
                ea.n = rows; ea.h = Hc + r0 * PS::P8; ea.pk = pkc + r0 * pkb; ea.t = tb->enc;
                if (!host_out) { ea.f = Fc + r0 * PS::P16; ea.ginv = Ic + r0 * PS::P16; ea.sk = skc + r0 * skb; }
                ProfScope ps_(PC_ENCODE, (double)rows, s);
                encode_kernel<PS><<<(unsigned)((rows + 3) / 4), 128, 0, s>>>(ea);
            }
            LAUNCHED();
            if (host_out) {
                CK(cudaEventRecord(cs->comp[buf], s));
                CK(cudaStreamWaitEvent(cs->s, cs->comp[buf], 0));
                CK(cudaMemcpyAsync(pk_out + (c0 + r0) * pkb, pkc + r0 * pkb, rows * pkb, cudaMemcpyDeviceToHost, cs->s));
            }
        }
        n_rq += m;
        if (host_out) CK(cudaEventRecord(cs->copy[buf], cs->s));
        if ((rc = route_flush(s)) || (rc = route_flush(s3))) return rc;
        }
    for (int li = l0; li < nl; li++) {     // join the lanes into the caller's stream
        CK(cudaEventRecord(lj->end[li], lanes[li].s));
        CK(cudaStreamWaitEvent(s0, lj->end[li], 0));
    }
    const bool async_host = host_out && (o.flags & SNTRUP_OPT_ASYNC) && o.done_event && !o.stats_out;
    if (host_out && !async_host) {         // join the copies into the caller's stream
        for (int li = 0; li < nl; li++)
            for (int i = 0; i < 2; i++) CK(cudaStreamWaitEvent(s0, csl[li]->copy[i], 0));
    }
    if (async_host) {
        // completion of every output byte, off the caller's stream: a side stream waits for
        // the lanes' last work and every copy, then records the user's event
        cudaStream_t ds = nullptr;
        cudaEvent_t s0_end = nullptr;
        if ((rc = done_stream(&ds, &s0_end))) return rc;
        CK(cudaEventRecord(s0_end, s0));                 // the lanes are joined into s0 above
        CK(cudaStreamWaitEvent(ds, s0_end, 0));
        for (int li = 0; li < nl; li++)
            for (int i = 0; i < 2; i++) CK(cudaStreamWaitEvent(ds, csl[li]->copy[i], 0));
        CK(cudaEventRecord((cudaEvent_t)o.done_event, ds));
    }
    {   // where this call's error flags live, for sntrup_async_error(stream) after an async call
        auto &e = g_async_err[std::make_pair(dev, (uintptr_t)s0)];
        e.assign(nl, nullptr);
        for (int li = 0; li < nl; li++) e[li] = lanes[li].err;
    }
    const bool sync = !(o.flags & SNTRUP_OPT_ASYNC) || (host_out && !async_host) || o.stats_out;
    if (sync) {
        int herr[MAX_LANES] = {};
        unsigned long long hrep[MAX_LANES] = {};
        for (int li = 0; li < nl; li++) {
            CK(cudaMemcpyAsync(&herr[li], lanes[li].err, sizeof(int), cudaMemcpyDeviceToHost, s0));
            CK(cudaMemcpyAsync(&hrep[li], lanes[li].repaired, sizeof(unsigned long long), cudaMemcpyDeviceToHost, s0));
        }
        CK(cudaStreamSynchronize(s0));
        for (int li = 0; li < nl; li++)
            if (herr[li]) return SNTRUP_E_INTERNAL;
        if (o.stats_out) {
            o.stats_out[0] = n_rq;
            o.stats_out[1] = n_r3;
            o.stats_out[2] = n_inv;
            o.stats_out[3] = hrep[0] + hrep[1] + hrep[2] + hrep[3];
        }
    }
    return SNTRUP_OK;
}

// ------------------------------------------------------------------------------ CUDA graphs
// SNTRUP_OPT_GRAPH: a keygen call's launches (every stream of the call: lanes, ring and aux
// streams fork from and join into the caller's stream) are captured once per call shape into a
// CUDA graph and replayed; the seed and first key index -- the only per-call values the kernels
// read besides the shape -- are patched into the captured sampler / repair kernel nodes.  For
// launch-bound calls (configs[0]: 32 keys) this removes the host enqueue and the inter-stream
// dependency latency from the call.
struct GraphKey {
    int dev, p;
    uint64_t n, chunk;
    uint32_t B, flags;
    uintptr_t stream, pk, sk, h, g, f, ginv, att, ws;
    size_t wsb;
    auto tie() const { return std::tie(dev, p, n, chunk, B, flags, stream, pk, sk, h, g, f, ginv, att, ws, wsb); }
    bool operator<(const GraphKey &o) const { return tie() < o.tie(); }
};
struct GraphArgNode {
    cudaGraphNode_t node;
    cudaKernelNodeParams prm;
    int kind;                     // 1 sampler, 2 repair
    uint64_t first_rel;           // the node's first key index - the call's
    SampleArgs sa;
    RepairArgs ra;
};
struct KeygenGraph {
    cudaGraph_t graph = nullptr;
    cudaGraphExec_t exec = nullptr;
    uint64_t epoch = 0;
    uint64_t kernels = 0;
    uint64_t last_use = 0;                  // g_graph_tick of the last capture / replay (LRU eviction)
    std::vector<GraphArgNode> nodes;
    std::vector<int *> errs;
};
inline std::map<GraphKey, KeygenGraph> g_graphs;
inline uint64_t g_graph_tick = 0;
// A graph is cached per call shape INCLUDING the output pointers; a caller that rotates through many
// output buffers would otherwise accumulate executable graphs without bound.
constexpr size_t MAX_GRAPHS = 32;

inline void graph_destroy(KeygenGraph &G) {
    if (G.exec) cudaGraphExecDestroy(G.exec);
    if (G.graph) cudaGraphDestroy(G.graph);
    G.exec = nullptr;
    G.graph = nullptr;
}
inline void graphs_release(uintptr_t stream = 0, bool all = true) {
    for (auto it = g_graphs.begin(); it != g_graphs.end();) {
        if (all || it->first.stream == stream) {
            graph_destroy(it->second);
            it = g_graphs.erase(it);
        } else {
            ++it;
        }
    }
}

// the synchronous tail of a keygen call (as keygen_impl's): the lanes' error flags
inline int keygen_finish(const sntrup_keygen_opts &o, const std::vector<int *> &errs, cudaStream_t s0) {
    if (o.flags & SNTRUP_OPT_ASYNC) return SNTRUP_OK;
    int herr[MAX_LANES] = {};
    for (size_t li = 0; li < errs.size() && li < (size_t)MAX_LANES; li++)
        CK(cudaMemcpyAsync(&herr[li], errs[li], sizeof(int), cudaMemcpyDeviceToHost, s0));
    CK(cudaStreamSynchronize(s0));
    for (size_t li = 0; li < errs.size() && li < (size_t)MAX_LANES; li++)
        if (herr[li]) return SNTRUP_E_INTERNAL;
    return SNTRUP_OK;
}

template <class PS>
int keygen_graph_host(uint64_t n, uint64_t seed, uint8_t *pk_out, uint8_t *sk_out, const sntrup_keygen_opts &o);

template <class PS>
int keygen_graph(uint64_t n, uint64_t seed, uint8_t *pk_out, uint8_t *sk_out, const sntrup_keygen_opts &o) {
    if (o.flags & SNTRUP_OPT_HOST_OUTPUT) return keygen_graph_host<PS>(n, seed, pk_out, sk_out, o);
    // device outputs on a non-default stream; no per-call host state (stats, host outputs)
    if ((o.flags & SNTRUP_OPT_SERIAL) || o.stats_out || o.done_event || !o.stream)
        return SNTRUP_E_ARG;
    int dev;
    CK(cudaGetDevice(&dev));
    const cudaStream_t s0 = (cudaStream_t)o.stream;
    sntrup_keygen_opts oa = o;
    oa.flags = (o.flags & ~SNTRUP_OPT_GRAPH) | SNTRUP_OPT_ASYNC;
    const GraphKey key{dev, PS::P, n, o.chunk_keys, o.batch_size, o.flags, (uintptr_t)s0, (uintptr_t)pk_out,
                       (uintptr_t)sk_out, (uintptr_t)o.h_out, (uintptr_t)o.g_out, (uintptr_t)o.f_out,
                       (uintptr_t)o.ginv_out, (uintptr_t)o.attempts_out, (uintptr_t)o.workspace, o.workspace_bytes};
    auto it = g_graphs.find(key);
    if (it != g_graphs.end() && it->second.epoch != g_ws_epoch) {      // workspace moved: rebuild
        graph_destroy(it->second);
        g_graphs.erase(it);
        it = g_graphs.end();
    }
    if (it == g_graphs.end()) {
        // first call of this shape: run it (reserves the workspace, produces this call's keys),
        // then capture the same enqueue sequence without executing it
        int rc = keygen_impl<PS>(n, seed, pk_out, sk_out, oa);
        if (rc) return rc;
        const std::vector<int *> errs = g_async_err[std::make_pair(dev, (uintptr_t)s0)];
        const uint64_t epoch = g_ws_epoch;
        const uint64_t l0 = g_launches.load();
        CK(cudaStreamBeginCapture(s0, cudaStreamCaptureModeThreadLocal));
        const int rc2 = keygen_impl<PS>(n, seed, pk_out, sk_out, oa);
        cudaGraph_t graph = nullptr;
        const cudaError_t ce = cudaStreamEndCapture(s0, &graph);
        g_launches.store(l0);
        if (rc2 || ce != cudaSuccess || !graph || g_ws_epoch != epoch) {
            if (graph) cudaGraphDestroy(graph);
            cudaGetLastError();
            return rc2 ? rc2 : SNTRUP_E_CUDA;
        }
        KeygenGraph G;
        G.graph = graph;
        G.epoch = epoch;
        G.errs = errs;
        if (cudaGraphInstantiate(&G.exec, graph, 0) != cudaSuccess) {
            graph_destroy(G);
            cudaGetLastError();
            return SNTRUP_E_CUDA;
        }
        // a failure past this point must not leak the instantiated graph
#define GCK(x) do { if ((x) != cudaSuccess) { graph_destroy(G); cudaGetLastError(); return SNTRUP_E_CUDA; } } while (0)
        size_t nn = 0;
        GCK(cudaGraphGetNodes(graph, nullptr, &nn));
        std::vector<cudaGraphNode_t> nodes(nn);
        GCK(cudaGraphGetNodes(graph, nodes.data(), &nn));
        for (cudaGraphNode_t nd : nodes) {
            cudaGraphNodeType t;
            GCK(cudaGraphNodeGetType(nd, &t));
            if (t != cudaGraphNodeTypeKernel) continue;
            G.kernels++;
            GraphArgNode a{};
            a.node = nd;
            GCK(cudaGraphKernelNodeGetParams(nd, &a.prm));
            if (a.prm.func == (void *)sample_kernel<PS>) {
                a.kind = 1;
                a.sa = *(const SampleArgs *)a.prm.kernelParams[0];
                if (a.sa.seed != seed) { graph_destroy(G); return SNTRUP_E_INTERNAL; }
                a.first_rel = a.sa.first - o.first_key_index;
            } else if (a.prm.func == (void *)repair_kernel<PS>) {
                a.kind = 2;
                a.ra = *(const RepairArgs *)a.prm.kernelParams[0];
                if (a.ra.seed != seed) { graph_destroy(G); return SNTRUP_E_INTERNAL; }
                a.first_rel = a.ra.first - o.first_key_index;
            } else {
                continue;
            }
            G.nodes.push_back(a);
        }
#undef GCK
        if (g_graphs.size() >= MAX_GRAPHS) {                 // evict the least recently used shape
            auto lru = g_graphs.begin();
            for (auto jt = g_graphs.begin(); jt != g_graphs.end(); ++jt)
                if (jt->second.last_use < lru->second.last_use) lru = jt;
            // a replay of it may still be running (its exec must outlive the launch), and its
            // stream may be gone by now: wait for the device, not for that stream
            if (cudaDeviceSynchronize() != cudaSuccess) cudaGetLastError();
            graph_destroy(lru->second);
            g_graphs.erase(lru);
        }
        G.last_use = ++g_graph_tick;
        g_graphs[key] = std::move(G);
        return keygen_finish(o, errs, s0);
    }
    KeygenGraph &G = it->second;
    G.last_use = ++g_graph_tick;
    for (GraphArgNode &a : G.nodes) {
        void *args[1];
        if (a.kind == 1) {
            a.sa.seed = seed;
            a.sa.first = o.first_key_index + a.first_rel;
            args[0] = &a.sa;
        } else {
            a.ra.seed = seed;
            a.ra.first = o.first_key_index + a.first_rel;
            args[0] = &a.ra;
        }
        cudaKernelNodeParams prm = a.prm;
        prm.kernelParams = args;
        prm.extra = nullptr;
        CK(cudaGraphExecKernelNodeSetParams(G.exec, a.node, &prm));
    }
    CK(cudaGraphLaunch(G.exec, s0));
    g_launches.fetch_add(G.kernels, std::memory_order_relaxed);
    g_async_err[std::make_pair(dev, (uintptr_t)s0)] = G.errs;
    return keygen_finish(o, G.errs, s0);
}

// SNTRUP_OPT_GRAPH | SNTRUP_OPT_HOST_OUTPUT | SNTRUP_OPT_ASYNC with a done event (the key-serving
// loop): the call is the graph replay of the device-output keygen into one of two whole-call
// output sets in device memory, followed by that set's two D2H copies on a copy stream, which
// then records the caller's event.  Why: while the previous call's 100 MB of pk/sk cross PCIe,
// every separately enqueued launch of this call starts later (the GPU fetches its commands over
// the same link: 2.55 -> 2.80 ms per 65,536-key call, scripts/serve_probe3.py); a graph launch is
// one submission and keeps 2.58 ms.  The copies of call k overlap the compute of call k+1 (two
// sets), not the call's own tail -- this mode is for back-to-back asynchronous calls.
struct GraphHost { cudaStream_t cs = nullptr; cudaEvent_t ready[2] = {}, copied[2] = {}; unsigned calls = 0; };
inline std::map<std::pair<int, uintptr_t>, GraphHost> g_graph_host;

template <class PS>
int keygen_graph_host(uint64_t n, uint64_t seed, uint8_t *pk_out, uint8_t *sk_out, const sntrup_keygen_opts &o) {
    if (!(o.flags & SNTRUP_OPT_ASYNC) || (o.flags & SNTRUP_OPT_SERIAL) || !o.done_event || o.stats_out || !o.stream)
        return SNTRUP_E_ARG;
    int dev;
    CK(cudaGetDevice(&dev));
    DevTables *tb;
    int rc = build_tables(dev, PS::P, PS::WT, &tb);
    if (rc) return rc;
    const size_t pkb = tb->enc.pk_bytes, skb = 2 * PS::SKH;
    const size_t set = align256(n * pkb) + align256(n * skb);
    const cudaStream_t s0 = (cudaStream_t)o.stream;
    GraphHost &gh = g_graph_host[std::make_pair(dev, (uintptr_t)s0)];
    if (!gh.cs) {
        if (make_stream(&gh.cs, -1)) return SNTRUP_E_CUDA;
        g_copy_streams.push_back(gh.cs);
        for (int i = 0; i < 2; i++) {
            CK(cudaEventCreateWithFlags(&gh.ready[i], cudaEventDisableTiming));
            CK(cudaEventCreateWithFlags(&gh.copied[i], cudaEventDisableTiming));
        }
    }
    char *base = nullptr;
    const uint64_t layout = ((uint64_t)PS::P << 48) ^ (n << 8) ^ 0xF;       // (the lanes' layouts end in nbuf, nl)
    if ((rc = staging_reserve(2 * set, layout, s0, &base))) return rc;
    const unsigned par = gh.calls++ & 1u;
    uint8_t *dpk = (uint8_t *)base + par * set, *dsk = dpk + align256(n * pkb);
    CK(cudaStreamWaitEvent(s0, gh.copied[par], 0));        // this set's previous copies (two calls ago)
    sntrup_keygen_opts od = o;
    od.flags = o.flags & ~SNTRUP_OPT_HOST_OUTPUT;
    od.done_event = nullptr;
    if ((rc = keygen_graph<PS>(n, seed, dpk, dsk, od))) return rc;
    CK(cudaEventRecord(gh.ready[par], s0));
    CK(cudaStreamWaitEvent(gh.cs, gh.ready[par], 0));
    CK(cudaMemcpyAsync(sk_out, dsk, n * skb, cudaMemcpyDeviceToHost, gh.cs));
    CK(cudaMemcpyAsync(pk_out, dpk, n * pkb, cudaMemcpyDeviceToHost, gh.cs));
    CK(cudaEventRecord(gh.copied[par], gh.cs));
    CK(cudaEventRecord((cudaEvent_t)o.done_event, gh.cs));
    return SNTRUP_OK;
}

// ------------------------------------------------------------------------------ small kernels
static __global__ void zero_rows_kernel(const int16_t *a, long long n, int p, long long stride,
                                 unsigned long long *first_zero) {
    const int lane = threadIdx.x & 31;
    const long long row = (long long)blockIdx.x * 4 + (threadIdx.x >> 5);
    if (row >= n) return;
    int nz = 0;
    for (int k = lane; k < p; k += 32) nz |= a[row * stride + k] != 0;
    nz = __any_sync(FULL, nz);
    if (!nz && lane == 0) atomicMin(first_zero, (unsigned long long)row);
}

// r3: small-factor test per element; G' = ok ? g : 1
template <class PS>
__global__ void __launch_bounds__(128) r3_prepare_kernel(const int8_t *g, int8_t *gp, uint8_t *ok_small,
                                                         long long n, const uint2 *T, const uint32_t *masks,
                                                         int nf) {
    constexpr int NBL = (PS::NB32 + 31) / 32;
    const int lane = threadIdx.x & 31;
    const long long row = (long long)blockIdx.x * 4 + (threadIdx.x >> 5);
    if (row >= n) return;
    uint32_t pl[NBL], mi[NBL];
#pragma unroll
    for (int s = 0; s < NBL; s++) {
        const int b = lane + 32 * s;
        if (b < PS::NB32) load_block_int8<PS>(g + row * PS::P16, b, pl[s], mi[s]);
        else { pl[s] = 0; mi[s] = 0; }
    }
    bool zero = true;
#pragma unroll
    for (int s = 0; s < NBL; s++) zero = zero && !(pl[s] | mi[s]);
    zero = __all_sync(FULL, zero);
    const bool sf = small_factor_check<PS, NBL>(pl, mi, T, masks, nf, lane);   // (always: constant time)
    const bool ok = !zero && sf;
#pragma unroll
    for (int s = 0; s < NBL; s++) {
        const int b = lane + 32 * s;
        if (32 * b < PS::P16)
            store_block_int8<PS>(gp + row * PS::P16, b, ok ? pl[s] : (b == 0 ? 1u : 0u), ok ? mi[s] : 0u);
    }
    if (lane == 0) ok_small[row] = ok ? 1 : 0;
}

// r3: finalize.  Trees whose root inverted: ok = ok_small (zero rows that were substituted).
// Trees whose root failed: exact per-element divstep on the original input.
// OUT = false (r3_is_invertible_batch): only ok[] is final; `out` is scratch written only for the
// rows of failed trees.
template <class PS, bool OUT = true>
__global__ void __launch_bounds__(128) r3_finalize_kernel(const int8_t *g, int8_t *out, uint8_t *ok,
                                                          long long n, int B, const uint8_t *root_ok) {
    const int lane = threadIdx.x & 31;
    const long long row = (long long)blockIdx.x * 4 + (threadIdx.x >> 5);
    if (row >= n) return;
    int8_t *orow = out + row * PS::P16;
    if (root_ok[row / B]) {
        if (OUT && !ok[row])
            for (int k = lane; k < PS::P16; k += 32) orow[k] = 0;
        return;
    }
    const bool inv = R3Divstep<PS>::invert(g + row * PS::P16, orow, lane);
    for (int k = PS::P + lane; k < PS::P16; k += 32) orow[k] = 0;
    if (lane == 0) ok[row] = inv ? 1 : 0;
}

template <class PS>
int r3_recip_impl(uint64_t n, const int8_t *g, int8_t *out, uint8_t *ok, uint32_t B_, cudaStream_t s) {
    int dev;
    CK(cudaGetDevice(&dev));
    DevTables *tb;
    int rc = build_tables(dev, PS::P, PS::WT, &tb);
    if (rc) return rc;
    const int B = B_ ? (int)B_ : 32;
    if (B < 1 || B > 4096 || (B & (B - 1))) return SNTRUP_E_ARG;
    const TreePlan tp = make_plan((long long)n, B);
    const long long inner = tp.inner_rows();
    size_t need = align256(n * PS::P16) + 2 * align256(inner * PS::P16 + 256 * (tp.L + 1)) +
                  align256(tp.cnt[tp.L]) + 4096;
    if ((rc = ws_reserve(need, s))) return rc;
    int8_t *gp = ws_take<int8_t>(n * PS::P16);
    std::vector<void *> l3(tp.L + 1, nullptr), i3(tp.L + 1, nullptr);
    for (int l = 1; l <= tp.L; l++) {
        l3[l] = ws_take<int8_t>(tp.cnt[l] * PS::P16);
        i3[l] = ws_take<int8_t>(tp.cnt[l] * PS::P16);
    }
    uint8_t *rok = ws_take<uint8_t>(tp.cnt[tp.L]);
    r3_prepare_kernel<PS><<<(unsigned)((n + 3) / 4), 128, 0, s>>>(g, gp, ok, (long long)n, tb->T, tb->masks, tb->nf);
    LAUNCHED();
    uint64_t np = 0;
    if ((rc = batch_inverse<PS, 3>(tp, rows8(gp, PS::P16), out, 1, PS::P16, l3, i3, rok, false, s, &np)))
        return rc;
    r3_finalize_kernel<PS><<<(unsigned)((n + 3) / 4), 128, 0, s>>>(g, out, ok, (long long)n, B, rok);
    LAUNCHED();
    CK(cudaStreamSynchronize(s));
    return SNTRUP_OK;
}

// isInvertible without the reciprocals: the small-factor residues decide the small
// factors; a tree's root (the product of its prepared leaves) is invertible iff every leaf is
// prime to the big factors, so only the up-sweep and the root divsteps run, and the leaves of a
// failed tree get their own divstep (invertibility only).  No down-sweep, no allocation.
template <class PS>
int r3_isinv_impl(uint64_t n, const int8_t *g, uint8_t *ok, cudaStream_t s) {
    int dev;
    CK(cudaGetDevice(&dev));
    DevTables *tb;
    int rc = build_tables(dev, PS::P, PS::WT, &tb);
    if (rc) return rc;
    const int B = 32;
    const TreePlan tp = make_plan((long long)n, B);
    size_t need = 2 * align256(n * PS::P16) + align256(tp.cnt[tp.L]);
    for (int l = 1; l <= tp.L; l++) need += 2 * align256(tp.cnt[l] * PS::P16);
    if ((rc = ws_reserve(need, s))) return rc;
    int8_t *gp = ws_take<int8_t>(n * PS::P16);
    int8_t *scratch = ws_take<int8_t>(n * PS::P16);
    std::vector<void *> l3(tp.L + 1, nullptr), i3(tp.L + 1, nullptr);
    for (int l = 1; l <= tp.L; l++) {
        l3[l] = ws_take<int8_t>(tp.cnt[l] * PS::P16);
        i3[l] = ws_take<int8_t>(tp.cnt[l] * PS::P16);
    }
    uint8_t *rok = ws_take<uint8_t>(tp.cnt[tp.L]);
    if (!ws_fits()) return SNTRUP_E_INTERNAL;
    {
        ProfScope ps_(PC_MISC, (double)n, s);              // (timed separately: tests of constant time)
        r3_prepare_kernel<PS><<<(unsigned)((n + 3) / 4), 128, 0, s>>>(g, gp, ok, (long long)n, tb->T, tb->masks, tb->nf);
    }
    LAUNCHED();
    const TreeJob<PS, 3> j{tp, rows8(gp, PS::P16), scratch, 1, PS::P16, l3, i3, rok, false};
    uint64_t np = 0;
    if ((rc = j.up(s, &np))) return rc;
    if ((rc = launch_divstep<PS, 3>(j.roots(), s))) return rc;
    r3_finalize_kernel<PS, false><<<(unsigned)((n + 3) / 4), 128, 0, s>>>(g, scratch, ok, (long long)n, B, rok);
    LAUNCHED();
    CK(cudaStreamSynchronize(s));
    return SNTRUP_OK;
}

template <class PS>
int rq_recip_impl(uint64_t n, const int16_t *a, int16_t *out, uint32_t B_, uint64_t *bad, cudaStream_t s) {
    const int B = B_ ? (int)B_ : 32;
    if (B < 1 || B > 4096 || (B & (B - 1))) return SNTRUP_E_ARG;
    const TreePlan tp = make_plan((long long)n, B);
    const long long inner = tp.inner_rows();
    size_t need = 2 * align256(inner * PS::P8 * 2 + 256 * (tp.L + 1)) + align256(tp.cnt[tp.L]) + 4096;
    int rc;
    if ((rc = ws_reserve(need, s))) return rc;
    std::vector<void *> lq(tp.L + 1, nullptr), iq(tp.L + 1, nullptr);
    for (int l = 1; l <= tp.L; l++) {
        lq[l] = ws_take<int16_t>(tp.cnt[l] * PS::P8);
        iq[l] = ws_take<int16_t>(tp.cnt[l] * PS::P8);
    }
    uint8_t *rok = ws_take<uint8_t>(tp.cnt[tp.L]);
    unsigned long long *fz = ws_take<unsigned long long>(1);
    CK(cudaMemsetAsync(fz, 0xff, sizeof(unsigned long long), s));
    zero_rows_kernel<<<(unsigned)((n + 3) / 4), 128, 0, s>>>(a, (long long)n, PS::P, PS::P8, fz);
    LAUNCHED();
    unsigned long long hz = 0;
    CK(cudaMemcpyAsync(&hz, fz, sizeof(hz), cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    if (hz != ~0ull) {
        if (bad) *bad = hz;
        return SNTRUP_E_NOT_INVERTIBLE;
    }
    uint64_t np = 0;
    if ((rc = batch_inverse<PS, PS::Q>(tp, rows16(a, PS::P8), out, 2, PS::P8, lq, iq, rok, false, s, &np)))
        return rc;
    CK(cudaStreamSynchronize(s));
    return SNTRUP_OK;
}


// ------------------------------------------------------------------------------ per-set entry points
// Everything that instantiates kernels for a parameter set goes through PsOps<PS>, defined in
// ps_ops.cuh and explicitly instantiated once per set in ps_<p>.cu (capi.cu only declares it).
template <class PS>
struct PsOps {
    static int keygen(uint64_t n, uint64_t seed, uint8_t *pk, uint8_t *sk, const sntrup_keygen_opts &o);
    static int mul_q(MulArgs m, cudaStream_t s, int la, int lb);     // in R/q
    static int mul_3(MulArgs m, cudaStream_t s, int la, int lb);     // in R/3
    static int r3_recip(uint64_t n, const int8_t *g, int8_t *out, uint8_t *ok, uint32_t B, cudaStream_t s);
    static int r3_isinv(uint64_t n, const int8_t *g, uint8_t *ok, cudaStream_t s);
    static int rq_recip(uint64_t n, const int16_t *a, int16_t *out, uint32_t B, uint64_t *bad, cudaStream_t s);
    static int full_sk(const FullSkArgs &a, int pkb, int skb, cudaStream_t s);
    static int sample_short(uint64_t seed, uint64_t first, uint64_t n, uint64_t domain, int8_t *out, cudaStream_t s);
    static int sample_uniform(uint64_t seed, uint64_t first, uint64_t n, uint64_t domain, int16_t *out,
                              cudaStream_t s);
    static int weight_check(const int8_t *r, uint64_t n, uint8_t *ok, cudaStream_t s);
    static int encode(uint64_t n, const int16_t *h, uint8_t *pk, cudaStream_t s);
};

}  // namespace sntrup_rt
