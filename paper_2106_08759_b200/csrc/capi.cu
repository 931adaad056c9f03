// capi.cu -- the C ABI of libsntrup_gpu.so (include/sntrup_gpu.h): argument checks, the library
// lock, and dispatch by parameter set to PsOps<PS> (runtime.cuh; instantiated in ps_<p>.cu).
//
// BatchKeyGen (Algorithm 1) per chunk of keys (runtime.cuh keygen_impl):
//   sample (f, g + small-factor isInvertible, retries)          sample.cuh
//   R/3 batchInv: product-tree up-sweep, root divstep, down-sweep, repair of failed trees
//   R/q batchInv on [3f]: up-sweep, root divstep, down-sweep     tcmul.cuh, tc4mul.cuh, divstep.cuh
//   H = [g * fbar]                                                (bottom level re-associated)
//   encode pk, sk                                                 encode.cuh
#include "runtime.cuh"
#include "intpeak.cuh"

using namespace sntrup;
using namespace sntrup_rt;

extern "C" {

int sntrup_params(int param_set, int *p, int *q, int *w, int *p_pad16, int *p_pad8,
                  size_t *pk_bytes, size_t *sk_bytes) {
    ParamInfo pi;
    if (!param_info(param_set, &pi)) return SNTRUP_E_PARAM;
    if (p) *p = pi.p;
    if (q) *q = pi.q;
    if (w) *w = pi.w;
    if (p_pad16) *p_pad16 = pi.p16;
    if (p_pad8) *p_pad8 = pi.p8;
    if (pk_bytes) *pk_bytes = pi.pk;
    if (sk_bytes) *sk_bytes = pi.sk;
    return SNTRUP_OK;
}

const char *sntrup_strerror(int code) {
    switch (code) {
    case SNTRUP_OK: return "ok";
    case SNTRUP_E_PARAM: return "unknown parameter set";
    case SNTRUP_E_ARG: return "invalid argument";
    case SNTRUP_E_NOT_INVERTIBLE: return "element not invertible";
    case SNTRUP_E_CUDA: return "CUDA error";
    case SNTRUP_E_WORKSPACE: return "device allocation failed";
    case SNTRUP_E_INTERNAL: return "internal error (retry bound exceeded)";
    default: return "unknown error";
    }
}

int sntrup_batch_keygen_ex(int param_set, uint64_t n_keys, uint64_t seed, uint8_t *pk_out,
                           uint8_t *sk_out, const sntrup_keygen_opts *opt) {
    ParamInfo pi;
    if (!param_info(param_set, &pi)) return SNTRUP_E_PARAM;
    if (n_keys == 0 || !pk_out || !sk_out) return SNTRUP_E_ARG;
    sntrup_keygen_opts o{};
    if (opt) o = *opt;
    std::lock_guard<std::mutex> lk(g_mu);
    SNTRUP_DISPATCH(param_set, return PsOps<PS>::keygen(n_keys, seed, pk_out, sk_out, o));
    return SNTRUP_E_PARAM;
}

int sntrup_batch_keygen(int param_set, uint64_t n_keys, uint64_t seed, uint8_t *pk_out,
                        uint8_t *sk_out) {
    return sntrup_batch_keygen_ex(param_set, n_keys, seed, pk_out, sk_out, nullptr);
}

size_t sntrup_keygen_workspace_bytes(int param_set, uint64_t n_keys, uint32_t batch_size) {
    return sntrup_keygen_workspace_bytes_ex(param_set, n_keys, batch_size, 0, 0);
}

size_t sntrup_keygen_workspace_bytes_ex(int param_set, uint64_t n_keys, uint32_t batch_size, uint32_t flags,
                                        uint64_t chunk_keys) {
    ParamInfo pi;
    if (!param_info(param_set, &pi) || n_keys == 0) return 0;
    const int B = batch_size ? (int)batch_size : 32;
    if (B < 1 || B > 4096 || (B & (B - 1))) return 0;
    SNTRUP_DISPATCH(param_set, {
        const KeygenShape k = keygen_shape<PS>(n_keys, B, flags, chunk_keys, pi.pk);
        return k.ws_need;
    });
    return 0;
}

size_t sntrup_workspace_reserved_bytes(void *stream, int which) {
    std::lock_guard<std::mutex> lk(g_mu);
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) return 0;
    if (which == 1) {
        auto it = g_stmap.find(std::make_pair(dev, (uintptr_t)stream));
        return it == g_stmap.end() ? 0 : it->second.cap;
    }
    auto it = g_wsmap.find(std::make_pair(dev, (uintptr_t)stream));
    return it == g_wsmap.end() ? 0 : it->second.cap;
}

int rq_mul_batch(int param_set, uint64_t n, const int16_t *a, const int16_t *b, int16_t *c,
                 void *stream) {
    ParamInfo pi;
    if (!param_info(param_set, &pi)) return SNTRUP_E_PARAM;
    if (n == 0 || !a || !b || !c) return SNTRUP_E_ARG;
    MulArgs m{};
    m.mode = MUL_ZIP;
    m.n_out = (long long)n;
    m.X = RowDesc{a, pi.p8, 2, 1};
    m.Y = RowDesc{b, pi.p8, 2, 1};
    m.out = c;
    m.out_stride = pi.p8;
    m.out_bytes = 2;
    m.periodic = 1;
    std::lock_guard<std::mutex> lk(g_mu);             // launcher caches, profiler state
    SNTRUP_DISPATCH(param_set, return PsOps<PS>::mul_q(m, (cudaStream_t)stream, 2, 2));
    return SNTRUP_E_PARAM;
}

int rq_mul_small_batch(int param_set, uint64_t n, const int16_t *a, const int8_t *b, int16_t *c,
                       void *stream) {
    ParamInfo pi;
    if (!param_info(param_set, &pi)) return SNTRUP_E_PARAM;
    if (n == 0 || !a || !b || !c) return SNTRUP_E_ARG;
    MulArgs m{};
    m.mode = MUL_ZIP;
    m.n_out = (long long)n;
    m.X = RowDesc{a, pi.p8, 2, 1};
    m.Y = RowDesc{b, pi.p16, 1, 1};
    m.out = c;
    m.out_stride = pi.p8;
    m.out_bytes = 2;
    m.periodic = 0;
    std::lock_guard<std::mutex> lk(g_mu);             // launcher caches, profiler state
    SNTRUP_DISPATCH(param_set, return PsOps<PS>::mul_q(m, (cudaStream_t)stream, 2, 1));
    return SNTRUP_E_PARAM;
}

size_t sntrup_full_sk_bytes(int param_set) {
    size_t pkb = 0, skb = 0;
    int p = 0;
    if (sntrup_params(param_set, &p, nullptr, nullptr, nullptr, nullptr, &pkb, &skb)) return 0;
    return skb + pkb + (size_t)((p + 3) / 4) + 32;
}

int sntrup_full_sk_batch(int param_set, uint64_t n, uint64_t seed, uint64_t first_key_index,
                         const uint8_t *pk, const uint8_t *sk, uint8_t *sk_full, void *stream) {
    size_t pkb = 0, skb = 0;
    if (sntrup_params(param_set, nullptr, nullptr, nullptr, nullptr, nullptr, &pkb, &skb)) return SNTRUP_E_PARAM;
    if (n == 0 || !pk || !sk || !sk_full) return SNTRUP_E_ARG;
    FullSkArgs a{seed, first_key_index, n, pk, sk, sk_full};
    const cudaStream_t s = (cudaStream_t)stream;
    SNTRUP_DISPATCH(param_set, return PsOps<PS>::full_sk(a, (int)pkb, (int)skb, s));
    return SNTRUP_E_PARAM;
}

int sntrup_event_create(void **ev) {
    if (!ev) return SNTRUP_E_ARG;
    cudaEvent_t e = nullptr;
    CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    *ev = (void *)e;
    return SNTRUP_OK;
}

int sntrup_event_synchronize(void *ev) {
    if (!ev) return SNTRUP_E_ARG;
    CK(cudaEventSynchronize((cudaEvent_t)ev));
    return SNTRUP_OK;
}

int sntrup_event_query(void *ev) {
    if (!ev) return SNTRUP_E_ARG;
    const cudaError_t e = cudaEventQuery((cudaEvent_t)ev);
    if (e == cudaErrorNotReady) return 1;
    CK(e);
    return SNTRUP_OK;
}

void sntrup_event_destroy(void *ev) {
    if (ev) cudaEventDestroy((cudaEvent_t)ev);
}

int sntrup_sample_short_batch(int param_set, uint64_t n, uint64_t seed, uint64_t first_key_index,
                              uint64_t domain, int8_t *r_out, void *stream) {
    ParamInfo pi;
    if (!param_info(param_set, &pi)) return SNTRUP_E_PARAM;
    if (n == 0 || !r_out) return SNTRUP_E_ARG;
    SNTRUP_DISPATCH(param_set, return PsOps<PS>::sample_short(seed, first_key_index, n, domain, r_out,
                                                              (cudaStream_t)stream));
    return SNTRUP_E_PARAM;
}

int sntrup_sample_uniform_rq_batch(int param_set, uint64_t n, uint64_t seed, uint64_t first_key_index,
                                    uint64_t domain, int16_t *a_out, void *stream) {
    ParamInfo pi;
    if (!param_info(param_set, &pi)) return SNTRUP_E_PARAM;
    if (n == 0 || !a_out) return SNTRUP_E_ARG;
    SNTRUP_DISPATCH(param_set, return PsOps<PS>::sample_uniform(seed, first_key_index, n, domain, a_out,
                                                                (cudaStream_t)stream));
    return SNTRUP_E_PARAM;
}

int sntrup_encap_core_batch(int param_set, uint64_t n, const int16_t *h, const int8_t *r, int16_t *c,
                            void *stream) {
    ParamInfo pi;
    if (!param_info(param_set, &pi)) return SNTRUP_E_PARAM;
    if (n == 0 || !h || !r || !c) return SNTRUP_E_ARG;
    std::lock_guard<std::mutex> lk(g_mu);
    MulArgs m{};
    m.mode = MUL_ZIP;
    m.n_out = (long long)n;
    m.X = RowDesc{h, pi.p8, 2, 1};
    m.Y = RowDesc{r, pi.p16, 1, 1};
    m.out = c;
    m.out_stride = pi.p8;
    m.out_bytes = 2;
    m.round3 = 1;                                   // c = Round(h * r)
    SNTRUP_DISPATCH(param_set, return PsOps<PS>::mul_q(m, (cudaStream_t)stream, 2, 1));
    return SNTRUP_E_PARAM;
}

int sntrup_decap_core_batch(int param_set, uint64_t n, const int8_t *f, const int8_t *ginv,
                            const int16_t *c, int8_t *r_out, uint8_t *ok, void *stream) {
    ParamInfo pi;
    if (!param_info(param_set, &pi)) return SNTRUP_E_PARAM;
    if (n == 0 || !f || !ginv || !c || !r_out || !ok) return SNTRUP_E_ARG;
    std::lock_guard<std::mutex> lk(g_mu);
    cudaStream_t s = (cudaStream_t)stream;
    int rc;
    if ((rc = ws_reserve(align256(n * pi.p8 * 2) + 4096, s))) return rc;
    int16_t *e = ws_take<int16_t>(n * pi.p8);
    SNTRUP_DISPATCH(param_set, {
        MulArgs m{};                                 // e = 3f * c in R/q
        m.mode = MUL_ZIP;
        m.n_out = (long long)n;
        m.X = RowDesc{c, pi.p8, 2, 1};
        m.Y = RowDesc{f, pi.p16, 1, 3};
        m.out = e;
        m.out_stride = pi.p8;
        m.out_bytes = 2;
        if ((rc = PsOps<PS>::mul_q(m, s, 2, 1))) return rc;
        MulArgs m3{};                                // r' = (e mod 3) * (1/g) in R/3
        m3.mode = MUL_ZIP;
        m3.n_out = (long long)n;
        m3.X = RowDesc{e, pi.p8, 2, 1, 1};
        m3.Y = RowDesc{ginv, pi.p16, 1, 1};
        m3.out = r_out;
        m3.out_stride = pi.p16;
        m3.out_bytes = 1;
        if ((rc = PsOps<PS>::mul_3(m3, s, 1, 1))) return rc;
        return PsOps<PS>::weight_check(r_out, n, ok, s);
    });
    return SNTRUP_E_PARAM;
}

int r3_mul_batch(int param_set, uint64_t n, const int8_t *a, const int8_t *b, int8_t *c,
                 void *stream) {
    ParamInfo pi;
    if (!param_info(param_set, &pi)) return SNTRUP_E_PARAM;
    if (n == 0 || !a || !b || !c) return SNTRUP_E_ARG;
    MulArgs m{};
    m.mode = MUL_ZIP;
    m.n_out = (long long)n;
    m.X = RowDesc{a, pi.p16, 1, 1};
    m.Y = RowDesc{b, pi.p16, 1, 1};
    m.out = c;
    m.out_stride = pi.p16;
    m.out_bytes = 1;
    m.periodic = 0;
    std::lock_guard<std::mutex> lk(g_mu);             // launcher caches, profiler state
    SNTRUP_DISPATCH(param_set, return PsOps<PS>::mul_3(m, (cudaStream_t)stream, 1, 1));
    return SNTRUP_E_PARAM;
}

int rq_recip_batch(int param_set, uint64_t n, const int16_t *a, int16_t *out, uint32_t batch_size,
                   uint64_t *bad_index, void *stream) {
    ParamInfo pi;
    if (!param_info(param_set, &pi)) return SNTRUP_E_PARAM;
    if (n == 0 || !a || !out) return SNTRUP_E_ARG;
    std::lock_guard<std::mutex> lk(g_mu);
    SNTRUP_DISPATCH(param_set, return PsOps<PS>::rq_recip(n, a, out, batch_size, bad_index, (cudaStream_t)stream));
    return SNTRUP_E_PARAM;
}

int r3_recip_batch(int param_set, uint64_t n, const int8_t *g, int8_t *out, uint8_t *ok,
                   uint32_t batch_size, void *stream) {
    ParamInfo pi;
    if (!param_info(param_set, &pi)) return SNTRUP_E_PARAM;
    if (n == 0 || !g || !out || !ok) return SNTRUP_E_ARG;
    std::lock_guard<std::mutex> lk(g_mu);
    SNTRUP_DISPATCH(param_set, return PsOps<PS>::r3_recip(n, g, out, ok, batch_size, (cudaStream_t)stream));
    return SNTRUP_E_PARAM;
}

int r3_is_invertible_batch(int param_set, uint64_t n, const int8_t *g, uint8_t *ok, void *stream) {
    ParamInfo pi;
    if (!param_info(param_set, &pi)) return SNTRUP_E_PARAM;
    if (n == 0 || !g || !ok) return SNTRUP_E_ARG;
    std::lock_guard<std::mutex> lk(g_mu);
    SNTRUP_DISPATCH(param_set, return PsOps<PS>::r3_isinv(n, g, ok, (cudaStream_t)stream));
    return SNTRUP_E_PARAM;
}

int rq_encode_batch(int param_set, uint64_t n, const int16_t *h, uint8_t *pk, void *stream) {
    ParamInfo pi;
    if (!param_info(param_set, &pi)) return SNTRUP_E_PARAM;
    if (n == 0 || !h || !pk) return SNTRUP_E_ARG;
    std::lock_guard<std::mutex> lk(g_mu);
    SNTRUP_DISPATCH(param_set, return PsOps<PS>::encode(n, h, pk, (cudaStream_t)stream));
    return SNTRUP_E_PARAM;
}

void sntrup_release_workspace(void) {
    std::lock_guard<std::mutex> lk(g_mu);
    int cur = 0;
    cudaGetDevice(&cur);
    for (auto &kv : g_wsmap) {
        if (!kv.second.base) continue;
        cudaSetDevice(kv.second.dev);
        cudaDeviceSynchronize();
        cudaFree(kv.second.base);
        kv.second.base = nullptr;
        kv.second.cap = 0;
    }
    for (cudaStream_t cs : g_copy_streams) cudaStreamSynchronize(cs);
    for (auto &kv : g_stmap) {
        if (!kv.second.base) continue;
        cudaSetDevice(kv.first.first);
        cudaFree(kv.second.base);
        kv.second.base = nullptr;
        kv.second.cap = 0;
    }
    cudaSetDevice(cur);
    g_ws = nullptr;
    ++g_ws_epoch;
    graphs_release();
}

int sntrup_release_stream_workspace(void *stream) {
    std::lock_guard<std::mutex> lk(g_mu);
    int dev = 0;
    CK(cudaGetDevice(&dev));
    const auto key = std::make_pair(dev, (uintptr_t)stream);
    CK(cudaStreamSynchronize((cudaStream_t)stream));
    for (cudaStream_t cs : g_copy_streams) CK(cudaStreamSynchronize(cs));
    graphs_release((uintptr_t)stream, false);
    ++g_ws_epoch;
    auto it = g_wsmap.find(key);
    if (it != g_wsmap.end() && it->second.base) {
        // the workspace held secret f, 1/g and tree rows: erase before freeing
        CK(cudaMemset(it->second.base, 0, it->second.cap));
        CK(cudaFree(it->second.base));
        if (g_ws == &it->second) g_ws = nullptr;
        g_wsmap.erase(it);
    }
    auto st = g_stmap.find(key);
    if (st != g_stmap.end() && st->second.base) {
        CK(cudaMemset(st->second.base, 0, st->second.cap));
        CK(cudaFree(st->second.base));
        g_stmap.erase(st);
    }
    return SNTRUP_OK;
}

int sntrup_measure_int_peak(int op, double *lane_ops_per_clk_sm, double *lane_ops_per_s) {
    if (op < 0 || op >= IOP_N) return SNTRUP_E_ARG;
    std::lock_guard<std::mutex> lk(g_mu);
    constexpr int CH = 8, ITER = 2048, NT = 256;
    const int sms = dev_info().sms, nb = sms * 8;
    uint32_t *sink = nullptr;
    IntPeakRec *rec = nullptr;
    CK(cudaMalloc(&sink, NT * sizeof(uint32_t)));
    CK(cudaMalloc(&rec, nb * sizeof(IntPeakRec)));
    cudaEvent_t e0, e1;
    CK(cudaEventCreate(&e0));
    CK(cudaEventCreate(&e1));
    auto launch = [&](cudaStream_t s) {
        switch (op) {
        case IOP_IMAD: int_peak_kernel<IOP_IMAD, CH, ITER><<<nb, NT, 0, s>>>(7u, sink, rec); break;
        case IOP_IADD3: int_peak_kernel<IOP_IADD3, CH, ITER><<<nb, NT, 0, s>>>(7u, sink, rec); break;
        case IOP_LOP3: int_peak_kernel<IOP_LOP3, CH, ITER><<<nb, NT, 0, s>>>(7u, sink, rec); break;
        default: int_peak_kernel<IOP_SHF, CH, ITER><<<nb, NT, 0, s>>>(7u, sink, rec); break;
        }
    };
    launch(0);                                   // warm-up (clocks up)
    LAUNCHED();
    CK(cudaEventRecord(e0, 0));
    launch(0);
    LAUNCHED();
    CK(cudaEventRecord(e1, 0));
    CK(cudaEventSynchronize(e1));
    float ms = 0;
    CK(cudaEventElapsedTime(&ms, e0, e1));
    std::vector<IntPeakRec> h(nb);
    CK(cudaMemcpy(h.data(), rec, nb * sizeof(IntPeakRec), cudaMemcpyDeviceToHost));
    cudaFree(sink);
    cudaFree(rec);
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    const double per_block = (double)NT * ITER * 8 * CH;
    std::map<unsigned, std::tuple<unsigned long long, unsigned long long, int>> sm;   // smid -> t0, t1, blocks
    for (auto &r : h) {
        auto it = sm.find(r.smid);
        if (it == sm.end()) sm[r.smid] = std::make_tuple(r.t0, r.t1, 1);
        else {
            auto &t = it->second;
            if (r.t0 < std::get<0>(t)) std::get<0>(t) = r.t0;
            if (r.t1 > std::get<1>(t)) std::get<1>(t) = r.t1;
            std::get<2>(t) += 1;
        }
    }
    double rate = 0;
    for (auto &kv : sm) rate += per_block * std::get<2>(kv.second) / (double)(std::get<1>(kv.second) - std::get<0>(kv.second));
    if (lane_ops_per_clk_sm) *lane_ops_per_clk_sm = sm.empty() ? 0 : rate / sm.size();
    if (lane_ops_per_s) *lane_ops_per_s = per_block * nb / (ms * 1e-3);
    return SNTRUP_OK;
}

int sntrup_ws_trace_read(int reset, uint64_t *out, int n) {
#ifdef SNTRUP_WS_TRACE
    std::lock_guard<std::mutex> lk(g_mu);
    constexpr size_t NB = 160 * 16 * sizeof(unsigned long long);
    if (!g_ws_trace) {
        CK(cudaMalloc(&g_ws_trace, NB));
        CK(cudaMemset(g_ws_trace, 0, NB));
    }
    CK(cudaDeviceSynchronize());
    static unsigned long long h[160 * 16];
    CK(cudaMemcpy(h, g_ws_trace, NB, cudaMemcpyDeviceToHost));
    for (int i = 0; i < n && i < 160 * 16; i++) out[i] = h[i];
    if (reset) CK(cudaMemset(g_ws_trace, 0, NB));
    return 160 * 16;
#else
    (void)reset; (void)out; (void)n;
    return 0;
#endif
}

uint64_t sntrup_kernel_launch_count(void) { return g_launches.load(); }

int sntrup_profile_read_kinds(int reset, double *ms, double *ops, uint64_t *launches) {
    std::lock_guard<std::mutex> lk(g_mu);
    prof_drain();
    for (int i = 0; i < PK_N; i++) {
        if (ms) ms[i] = g_kagg[i].ms;
        if (ops) ops[i] = g_kagg[i].ops;
        if (launches) launches[i] = g_kagg[i].launches;
    }
    if (reset)
        for (int i = 0; i < PK_N; i++) g_kagg[i] = ProfAgg{};
    return PK_N;
}

int sntrup_profile_read_kinds_ex(int reset, double *ms, double *ops, uint64_t *launches, double *products,
                                 double *smem_bytes) {
    std::lock_guard<std::mutex> lk(g_mu);
    prof_drain();
    for (int i = 0; i < PK_N; i++) {
        if (ms) ms[i] = g_kagg[i].ms;
        if (ops) ops[i] = g_kagg[i].ops;
        if (launches) launches[i] = g_kagg[i].launches;
        if (products) products[i] = g_kagg[i].units;
        if (smem_bytes) smem_bytes[i] = g_kagg[i].smem;
    }
    if (reset)
        for (int i = 0; i < PK_N; i++) g_kagg[i] = ProfAgg{};
    return PK_N;
}

int sntrup_async_error(void *stream) {
    std::lock_guard<std::mutex> lk(g_mu);
    int dev = 0;
    CK(cudaGetDevice(&dev));
    auto it = g_async_err.find(std::make_pair(dev, (uintptr_t)stream));
    if (it == g_async_err.end()) return SNTRUP_OK;
    CK(cudaStreamSynchronize((cudaStream_t)stream));
    for (int *e : it->second) {
        int h = 0;
        CK(cudaMemcpy(&h, e, sizeof(int), cudaMemcpyDeviceToHost));
        if (h) return SNTRUP_E_INTERNAL;
    }
    return SNTRUP_OK;
}

int sntrup_set_divstep_threads(int nt) {
    if (nt != 128 && nt != 256 && nt != 512 && nt != 768) return SNTRUP_E_ARG;
    std::lock_guard<std::mutex> lk(g_mu);
    g_divstep_threads = nt;
    return SNTRUP_OK;
}

int sntrup_set_root_impl(int impl) {
    if (impl < 0 || impl > 7 || (impl & 3) == 3) return SNTRUP_E_ARG;
    std::lock_guard<std::mutex> lk(g_mu);
    g_root_impl = impl;
    return SNTRUP_OK;
}

int sntrup_set_sched(long long top_items, long long items_cap) {
    if (top_items < 0 || items_cap < 0) return SNTRUP_E_ARG;
    std::lock_guard<std::mutex> lk(g_mu);
    g_top_items = top_items;
    g_items_cap = items_cap;
    return SNTRUP_OK;
}

int sntrup_set_mul_impl(int impl) {
    if (impl < 0 || impl > 16) return SNTRUP_E_ARG;
    std::lock_guard<std::mutex> lk(g_mu);
    g_mul_impl = impl;
    return SNTRUP_OK;
}

void sntrup_profile_enable(int on) {
    std::lock_guard<std::mutex> lk(g_mu);
    prof_drain();
    g_prof_on = on != 0;
}

int sntrup_profile_read(int reset, double *ms, double *units, double *ops, uint64_t *launches,
                        int max_classes) {
    std::lock_guard<std::mutex> lk(g_mu);
    prof_drain();
    const int n = max_classes < PC_N ? max_classes : PC_N;
    for (int i = 0; i < n; i++) {
        if (ms) ms[i] = g_agg[i].ms;
        if (units) units[i] = g_agg[i].units;
        if (ops) ops[i] = g_agg[i].ops;
        if (launches) launches[i] = g_agg[i].launches;
    }
    if (reset)
        for (int i = 0; i < PC_N; i++) g_agg[i] = ProfAgg{};
    return PC_N;
}

}  // extern "C"

