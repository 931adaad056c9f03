// ps_ops.cuh -- definitions of PsOps<PS> (runtime.cuh); included only by the per-parameter-set
// translation units ps_<p>.cu, each of which instantiates it for one set.
#pragma once
#include "runtime.cuh"

namespace sntrup_rt {

template <class PS>
int PsOps<PS>::keygen(uint64_t n, uint64_t seed, uint8_t *pk, uint8_t *sk, const sntrup_keygen_opts &o) {
    if (o.flags & SNTRUP_OPT_GRAPH) return keygen_graph<PS>(n, seed, pk, sk, o);
    return keygen_impl<PS>(n, seed, pk, sk, o);
}
template <class PS>
int PsOps<PS>::mul_q(MulArgs m, cudaStream_t s, int la, int lb) { return launch_mul<PS, PS::Q>(m, s, la, lb); }
template <class PS>
int PsOps<PS>::mul_3(MulArgs m, cudaStream_t s, int la, int lb) { return launch_mul<PS, 3>(m, s, la, lb); }
template <class PS>
int PsOps<PS>::r3_recip(uint64_t n, const int8_t *g, int8_t *out, uint8_t *ok, uint32_t B, cudaStream_t s) {
    return r3_recip_impl<PS>(n, g, out, ok, B, s);
}
template <class PS>
int PsOps<PS>::r3_isinv(uint64_t n, const int8_t *g, uint8_t *ok, cudaStream_t s) {
    return r3_isinv_impl<PS>(n, g, ok, s);
}
template <class PS>
int PsOps<PS>::rq_recip(uint64_t n, const int16_t *a, int16_t *out, uint32_t B, uint64_t *bad, cudaStream_t s) {
    return rq_recip_impl<PS>(n, a, out, B, bad, s);
}
template <class PS>
int PsOps<PS>::full_sk(const FullSkArgs &a, int pkb, int skb, cudaStream_t s) {
    full_sk_copy_kernel<PS><<<(unsigned)((a.n + 3) / 4), 128, 0, s>>>(a, pkb, skb);
    LAUNCHED();
    sha512_pk_kernel<PS><<<(unsigned)((a.n + 127) / 128), 128, 0, s>>>(a, pkb, skb);
    LAUNCHED();
    return SNTRUP_OK;
}
template <class PS>
int PsOps<PS>::sample_short(uint64_t seed, uint64_t first, uint64_t n, uint64_t domain, int8_t *out,
                            cudaStream_t s) {
    short_kernel<PS><<<(unsigned)((n + 3) / 4), 128, 0, s>>>(seed, first, n, domain, out);
    LAUNCHED();
    return SNTRUP_OK;
}
template <class PS>
int PsOps<PS>::sample_uniform(uint64_t seed, uint64_t first, uint64_t n, uint64_t domain, int16_t *out,
                              cudaStream_t s) {
    const uint64_t threads = n * (uint64_t)(PS::P8 / 2);
    uniform_rq_kernel<PS><<<(unsigned)((threads + 127) / 128), 128, 0, s>>>(seed, first, n, domain, out);
    LAUNCHED();
    return SNTRUP_OK;
}
template <class PS>
int PsOps<PS>::weight_check(const int8_t *r, uint64_t n, uint8_t *ok, cudaStream_t s) {
    weight_check_kernel<PS><<<(unsigned)((n + 3) / 4), 128, 0, s>>>(r, n, ok);
    LAUNCHED();
    return SNTRUP_OK;
}
template <class PS>
int PsOps<PS>::encode(uint64_t n, const int16_t *h, uint8_t *pk, cudaStream_t s) {
    int dev;
    CK(cudaGetDevice(&dev));
    DevTables *tb;
    int rc = build_tables(dev, PS::P, PS::WT, &tb);
    if (rc) return rc;
    EncArgs ea{};
    ea.n = n; ea.h = h; ea.pk = pk; ea.t = tb->enc;
    encode_kernel<PS><<<(unsigned)((n + 3) / 4), 128, 0, s>>>(ea);
    LAUNCHED();
    return SNTRUP_OK;
}

}  // namespace sntrup_rt
