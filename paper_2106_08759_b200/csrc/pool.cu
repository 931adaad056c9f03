// pool.cu -- GPU-backed key pool: the paper's engNTRU batch_lib provider (section
// 4.2) on B200.  The paper keeps a thread-safe pool of pre-generated key pairs per parameter set,
// filled lazily by one BatchKeyGen call and refilled when empty, so a TLS handshake's keygen
// becomes a memcpy ("first key 2.5 ms, then 0 ms").  Here the batches are
// sntrup_batch_keygen_ex calls on a private stream into device buffers, copied into a pinned host
// ring; take() hands out the next key pair (host copy + secure erase of the ring slot) and starts
// an asynchronous refill whenever the ready keys fall to half the capacity, so a steady consumer
// never waits for the GPU.  Keys carry consecutive global key indices of one seed, so every
// handed-out pair is reproducible by the oracle.
#include <condition_variable>
#include <cstdio>
#include <cstring>
#include <mutex>
#include <vector>

#include <cuda_runtime.h>

#include "../../include/sntrup_gpu.h"

struct sntrup_pool {
    int param_set = 0;
    uint64_t seed = 0, next_index = 0, batch = 0;
    uint32_t tree_b = 0;
    size_t pkb = 0, skb = 0;
    int nslots = 0;
    uint8_t *h_pk = nullptr, *h_sk = nullptr;      // pinned ring: nslots * batch keys
    uint8_t *d_pk = nullptr, *d_sk = nullptr;      // device: one batch
    cudaStream_t st = nullptr;
    enum { EMPTY = 0, FILLING = 1, READY = 2 };
    struct Slot { int state = EMPTY; cudaEvent_t ev = nullptr; uint64_t first = 0, taken = 0; };
    std::vector<Slot> slots;
    int head = 0, tail = 0;                        // head: oldest non-empty slot; tail: next to fill
    std::mutex mu;
    uint64_t n_taken = 0, n_generated = 0, n_waits = 0;
    int dev = 0;
};

namespace {

int pool_ck(cudaError_t e) {
    if (e != cudaSuccess) {
        fprintf(stderr, "sntrup_pool: %s\n", cudaGetErrorString(e));
        return SNTRUP_E_CUDA;
    }
    return SNTRUP_OK;
}

// Start filling slot `tail` (caller holds p->mu).  Returns SNTRUP_OK or an error.
int pool_refill(sntrup_pool *p) {
    sntrup_pool::Slot &s = p->slots[p->tail];
    if (s.state != sntrup_pool::EMPTY) return SNTRUP_OK;
    sntrup_keygen_opts o;
    memset(&o, 0, sizeof(o));
    o.first_key_index = p->next_index;
    o.batch_size = p->tree_b;
    o.flags = SNTRUP_OPT_ASYNC;
    o.stream = p->st;
    int rc = sntrup_batch_keygen_ex(p->param_set, p->batch, p->seed, p->d_pk, p->d_sk, &o);
    if (rc) return rc;
    const size_t off = (size_t)p->tail * p->batch;
    if ((rc = pool_ck(cudaMemcpyAsync(p->h_pk + off * p->pkb, p->d_pk, p->batch * p->pkb,
                                      cudaMemcpyDeviceToHost, p->st)))) return rc;
    if ((rc = pool_ck(cudaMemcpyAsync(p->h_sk + off * p->skb, p->d_sk, p->batch * p->skb,
                                      cudaMemcpyDeviceToHost, p->st)))) return rc;
    if ((rc = pool_ck(cudaEventRecord(s.ev, p->st)))) return rc;
    s.state = sntrup_pool::FILLING;
    s.first = p->next_index;
    s.taken = 0;
    p->next_index += p->batch;
    p->n_generated += p->batch;
    p->tail = (p->tail + 1) % p->nslots;
    return SNTRUP_OK;
}

uint64_t pool_ready_keys(sntrup_pool *p) {
    uint64_t r = 0;
    for (auto &s : p->slots)
        if (s.state != sntrup_pool::EMPTY) r += p->batch - s.taken;
    return r;
}

}  // namespace

extern "C" {

int sntrup_pool_create(int param_set, uint64_t seed, uint64_t first_key_index, uint64_t capacity,
                       uint64_t batch_keys, uint32_t batch_size, sntrup_pool **out) {
    if (!out) return SNTRUP_E_ARG;
    *out = nullptr;
    size_t pkb = 0, skb = 0;
    if (sntrup_params(param_set, nullptr, nullptr, nullptr, nullptr, nullptr, &pkb, &skb)) return SNTRUP_E_PARAM;
    if (batch_keys == 0 || capacity < 2 * batch_keys || capacity % batch_keys) return SNTRUP_E_ARG;
    sntrup_pool *p = new sntrup_pool();
    p->param_set = param_set;
    p->seed = seed;
    p->next_index = first_key_index;
    p->batch = batch_keys;
    p->tree_b = batch_size;
    p->pkb = pkb;
    p->skb = skb;
    p->nslots = (int)(capacity / batch_keys);
    p->slots.resize(p->nslots);
    cudaGetDevice(&p->dev);
    int rc = SNTRUP_OK;
    if (!rc) rc = pool_ck(cudaHostAlloc(&p->h_pk, capacity * pkb, cudaHostAllocDefault));
    if (!rc) rc = pool_ck(cudaHostAlloc(&p->h_sk, capacity * skb, cudaHostAllocDefault));
    if (!rc) rc = pool_ck(cudaMalloc(&p->d_pk, batch_keys * pkb));
    if (!rc) rc = pool_ck(cudaMalloc(&p->d_sk, batch_keys * skb));
    if (!rc) rc = pool_ck(cudaStreamCreateWithFlags(&p->st, cudaStreamNonBlocking));
    for (auto &s : p->slots)
        if (!rc) rc = pool_ck(cudaEventCreateWithFlags(&s.ev, cudaEventDisableTiming));
    if (rc) {
        sntrup_pool_destroy(p);
        return rc == SNTRUP_E_CUDA ? SNTRUP_E_WORKSPACE : rc;
    }
    *out = p;
    return SNTRUP_OK;
}

int sntrup_pool_take(sntrup_pool *p, uint8_t *pk, uint8_t *sk, uint64_t *key_index) {
    if (!p || !pk || !sk) return SNTRUP_E_ARG;
    std::lock_guard<std::mutex> lk(p->mu);
    int dev_save = 0;
    cudaGetDevice(&dev_save);
    cudaSetDevice(p->dev);
    int rc = SNTRUP_OK;
    sntrup_pool::Slot *s = &p->slots[p->head];
    if (s->state == sntrup_pool::EMPTY) {          // nothing generated yet: fill now (lazy fill)
        if ((rc = pool_refill(p))) goto done;
        s = &p->slots[p->head];
    }
    if (s->state == sntrup_pool::FILLING) {
        const cudaError_t q = cudaEventQuery(s->ev);
        if (q == cudaErrorNotReady) {
            p->n_waits++;
            if ((rc = pool_ck(cudaEventSynchronize(s->ev)))) goto done;
        } else if ((rc = pool_ck(q))) {
            goto done;
        }
        // the refill was asynchronous: check its device error flags (g retry bound) now
        if ((rc = sntrup_async_error(p->st))) goto done;
        s->state = sntrup_pool::READY;
    }
    {
        const size_t k = (size_t)p->head * p->batch + s->taken;
        memcpy(pk, p->h_pk + k * p->pkb, p->pkb);
        memcpy(sk, p->h_sk + k * p->skb, p->skb);
        memset(p->h_sk + k * p->skb, 0, p->skb);   // secure erase of the handed-out secret key
        memset(p->h_pk + k * p->pkb, 0, p->pkb);
        if (key_index) *key_index = s->first + s->taken;
        s->taken++;
        p->n_taken++;
        if (s->taken == p->batch) {
            s->state = sntrup_pool::EMPTY;
            p->head = (p->head + 1) % p->nslots;
        }
    }
    // keep the ring at least half full: one refill in flight at a time
    {
        bool filling = false;
        for (auto &x : p->slots) filling = filling || x.state == sntrup_pool::FILLING;
        if (!filling && pool_ready_keys(p) <= (uint64_t)p->nslots * p->batch / 2) rc = pool_refill(p);
    }
done:
    cudaSetDevice(dev_save);
    return rc;
}

int sntrup_pool_stats(sntrup_pool *p, uint64_t *taken, uint64_t *generated, uint64_t *waits,
                      uint64_t *ready) {
    if (!p) return SNTRUP_E_ARG;
    std::lock_guard<std::mutex> lk(p->mu);
    if (taken) *taken = p->n_taken;
    if (generated) *generated = p->n_generated;
    if (waits) *waits = p->n_waits;
    if (ready) *ready = pool_ready_keys(p);
    return SNTRUP_OK;
}

void sntrup_pool_destroy(sntrup_pool *p) {
    if (!p) return;
    int dev_save = 0;
    cudaGetDevice(&dev_save);
    cudaSetDevice(p->dev);
    if (p->st) {
        cudaStreamSynchronize(p->st);
        sntrup_release_stream_workspace(p->st);   // erase + free the keygen workspace of the pool's stream
    }
    if (p->h_sk) { memset(p->h_sk, 0, (size_t)p->nslots * p->batch * p->skb); cudaFreeHost(p->h_sk); }
    if (p->h_pk) cudaFreeHost(p->h_pk);
    if (p->d_pk) cudaFree(p->d_pk);
    if (p->d_sk) { cudaMemset(p->d_sk, 0, p->batch * p->skb); cudaFree(p->d_sk); }
    for (auto &s : p->slots)
        if (s.ev) cudaEventDestroy(s.ev);
    if (p->st) cudaStreamDestroy(p->st);
    cudaSetDevice(dev_save);
    delete p;
}

}  // extern "C"
