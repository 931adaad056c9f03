/*
 * sntrup_gpu.h -- C ABI of libsntrup_gpu.so: batched Streamlined NTRU Prime key generation and
 * the ring primitives it is built from, as hand-written CUDA kernels for sm_100a (B200).
 *
 * Paper: arXiv 2106.08759 ("OpenSSLNTRU").  "P:N" cites line N of its LaTeX source.
 *   KeyGen            P:3398-3461 (section 3.1): g small, invertible in R/3; f in Short;
 *                     h = g/(3f) in R/q; output (h, (f, 1/g)).
 *   BatchKeyGen       P:3597-3618 (Algorithm 1): the 2n inversions replaced by two batchInv.
 *   batchInv          P:1432-1561 (section 2.2): Montgomery's trick, 3n-3 multiplications and
 *                     one inversion for n inverses (here: level-parallel product trees).
 *   isInvertible      P:3620-4070 (section 3.1.1): g mod f_i != 0 for every factor f_i of
 *                     x^p - x - 1 over GF(3).
 *   Rings             P:1361-1385 (section 2.1): R/3 = (Z/3)[x]/(x^p-x-1), R/q = (Z/q)[x]/(x^p-x-1),
 *                     R/q a field; parameter sets P:1418-1430 plus 953/1013/1277 (Z20).
 *
 * Conventions ("readings"):
 *   - param_set is p, one of {653, 761, 857, 953, 1013, 1277}; anything else -> SNTRUP_E_PARAM.
 *   - R/q elements: int16 rows, coefficients centered in [-(q-1)/2, (q-1)/2], row stride
 *     p8 = 8*ceil(p/8) elements.  R/3 / Small / Short elements: int8 rows in {-1,0,1}, row stride
 *     p16 = 16*ceil(p/16) elements.  Pad lanes of inputs must be 0; pad lanes of outputs are
 *     written 0.  Inputs outside the canonical range are a precondition violation (unchecked).
 *   - pk = radix Rq-encode(h) (pk_bytes per key), sk = Small-encode(f) || Small-encode(1/g)
 *     (sk_bytes = 2*ceil(p/4) per key); row strides are pk_bytes / sk_bytes (dense).
 *   - Randomness: per-key SplitMix64 counter stream keyed by (seed, global key index), consumed
 *     in the documented order (C2-C4).  Outputs depend only on (param_set, seed,
 *     global key index): never on batch size, chunking or stream.
 *   - Pointers are CUDA device pointers unless stated; the caller owns every buffer.  Calls are
 *     stream-ordered on `stream` (NULL = legacy default stream) and return after enqueueing,
 *     except where "synchronous" is stated.  The library keeps an internal cached workspace
 *     (one per device and per stream) and constant tables; no other state.
 *   - Errors: negative return codes below; CUDA failures -> SNTRUP_E_CUDA.  No call aborts.
 */
#ifndef SNTRUP_GPU_H
#define SNTRUP_GPU_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum {
    SNTRUP_OK = 0,
    SNTRUP_E_PARAM = -1,          /* unknown param_set */
    SNTRUP_E_ARG = -2,            /* n == 0, NULL required pointer, bad batch size */
    SNTRUP_E_NOT_INVERTIBLE = -3, /* rq_recip_batch: some input is 0 (R/q is a field) */
    SNTRUP_E_CUDA = -4,           /* a CUDA runtime call failed */
    SNTRUP_E_WORKSPACE = -5,      /* device allocation failed */
    SNTRUP_E_INTERNAL = -6        /* retry bound exceeded (g never invertible) */
};

/* Parameters of a set.  Any output pointer may be NULL.  Returns SNTRUP_OK or
   SNTRUP_E_PARAM. */
int sntrup_params(int param_set, int *p, int *q, int *w, int *p_pad16, int *p_pad8,
                  size_t *pk_bytes, size_t *sk_bytes);

/* Human-readable name of an error code (static string). */
const char *sntrup_strerror(int code);

/* Batch key generation (Algorithm 1) of n_keys key pairs with global key indices
   0 .. n_keys-1 of stream `seed`, Montgomery batch size 32 (the paper's library default,
   P:7187-7200).  pk_out: uint8[n_keys][pk_bytes], sk_out: uint8[n_keys][sk_bytes], device
   pointers.  Synchronous (returns after the outputs are complete).  n_keys == 0 -> SNTRUP_E_ARG. */
int sntrup_batch_keygen(int param_set, uint64_t n_keys, uint64_t seed,
                        uint8_t *pk_out, uint8_t *sk_out);

/* Option flags for sntrup_keygen_opts.flags */
#define SNTRUP_OPT_HOST_OUTPUT    1u  /* pk_out/sk_out are HOST pointers (pinned recommended):
                                         the library copies each chunk back as it completes */
#define SNTRUP_OPT_NO_SMALL_CHECK 2u  /* test hook: skip the small-factor invertibility test in
                                         the sampler, so every non-invertible g is caught by the
                                         product-tree root check and repaired */
#define SNTRUP_OPT_ASYNC          4u  /* do not synchronise before returning (device outputs) */
#define SNTRUP_OPT_RING_STREAMS   16u /* run the R/3 tree chain on its own stream beside the R/q
                                         chain (separate root inversions) instead of one stream
                                         with a joint root launch; outputs identical */
#define SNTRUP_OPT_FORCE_SMALL_CHECK 8u /* always run the sampler's small-factor test (by default it
                                         is skipped where a tree almost never fails without it:
                                         B * P(small-factor rejection per draw) <= 1e-4,
                                         e.g. 761/857;
                                         outputs are identical either way) */
#define SNTRUP_OPT_LANES4         32u /* pipeline up to 4 chunks concurrently (one stream set per
                                         lane) instead of 2; outputs identical */
#define SNTRUP_OPT_STAGGER       128u /* lane k of the first round starts when lane k-1 has finished
                                         its R/q up-sweep (its throughput phases fill lane k-1's
                                         latency-bound root inversion); outputs identical */
#define SNTRUP_OPT_SERIAL        256u /* measurement: every kernel of the call on the caller's
                                         stream, one at a time (one lane, no ring / aux streams),
                                         so per-launch CUDA-event times are each kernel's own;
                                         outputs identical */
#define SNTRUP_OPT_LANE_PRIORITY  64u /* lanes on internal streams of decreasing priority: the
                                         first lane's chunk completes first (its D2H copies overlap
                                         the other lanes' compute); outputs identical */
#define SNTRUP_OPT_GRAPH         512u /* replay the call as a CUDA graph: the first call of a shape
                                         (param set, n, B, chunk, flags, stream, output / debug
                                         pointers, workspace) runs normally and then captures its
                                         launches on every stream of the call into a graph; later
                                         calls of that shape patch the seed and first key index into
                                         the captured sampler / repair kernels and launch the graph.
                                         Device outputs on a non-default stream (no stats or
                                         done_event: SNTRUP_E_ARG); the graph is
                                         rebuilt when the stream's workspace is reallocated and
                                         dropped by sntrup_release_[stream_]workspace.  Outputs
                                         identical; for launch-bound calls (configs[0]) it removes
                                         the host enqueue and inter-stream latency.
                                         With SNTRUP_OPT_HOST_OUTPUT (the key-serving loop): only
                                         together with SNTRUP_OPT_ASYNC and a done_event on a
                                         non-default stream (else SNTRUP_E_ARG).  The call replays
                                         the device-output graph into one of two whole-call output
                                         sets in device memory (2 n (pk + sk) bytes of staging),
                                         then copies that set to pk_out / sk_out on a copy stream
                                         and records done_event after the last byte; the copies of
                                         one call overlap the compute of the next.  A graph launch
                                         is one submission, so it is not slowed by the previous
                                         call's D2H traffic on the host link the way ~90 separate
                                         launches are (2.80 -> 2.58 ms per 65,536-key call). */

typedef struct {
    uint64_t first_key_index; /* keys first .. first+n-1 (chunked / resumable / multi-GPU runs) */
    uint32_t batch_size;      /* B = keys per product tree, power of two in [1, 4096]; 0 -> 32 */
    uint32_t flags;           /* SNTRUP_OPT_* */
    uint64_t chunk_keys;      /* keys per internal chunk (0 -> library default, 65536 rounded to B) */
    void *stream;             /* cudaStream_t; NULL -> legacy default stream */
    int16_t *h_out;           /* optional device [n][p8]: centered public h */
    int8_t *g_out;            /* optional device [n][p16]: accepted g */
    int8_t *f_out;            /* optional device [n][p16]: f */
    int8_t *ginv_out;         /* optional device [n][p16]: 1/g in R/3 */
    uint8_t *attempts_out;    /* optional device [n]: number of g draws used (>= 1) */
    uint64_t *stats_out;      /* optional HOST uint64[4]: ring products R/q, ring products R/3,
                                 root inversions, keys repaired (trees whose R/3 root failed) */
    void *done_event;         /* optional sntrup_event (sntrup_event_create): with
                                 SNTRUP_OPT_HOST_OUTPUT | SNTRUP_OPT_ASYNC the call returns after
                                 enqueueing, the outputs' D2H copies are NOT ordered into `stream`
                                 (the next call's compute overlaps them), and this event completes
                                 when every pk/sk byte is in host memory.  The host buffers must
                                 stay untouched until then. */
    void *workspace;          /* optional caller-owned DEVICE scratch (256-byte aligned) of
                                 workspace_bytes >= sntrup_keygen_workspace_bytes_ex(...) for this
                                 call's shape (else SNTRUP_E_WORKSPACE; misaligned -> SNTRUP_E_ARG);
                                 NULL -> the library's cached workspace of `stream`.  The caller
                                 keeps it alive and unused until the call's work has completed
                                 (host-output staging is separate and library-owned). */
    size_t workspace_bytes;
} sntrup_keygen_opts;

/* Error status of the last keygen call on `stream` (device pointers / SNTRUP_OPT_ASYNC calls do
   not read their device error flags before returning): synchronises `stream`, then
   SNTRUP_E_INTERNAL if that call hit the g retry bound, else SNTRUP_OK.  Valid until the next
   call on the stream. */
int sntrup_async_error(void *stream);

/* Completion events for asynchronous host-output calls (opaque cudaEvent_t). */
int sntrup_event_create(void **ev);
int sntrup_event_synchronize(void *ev);       /* blocks until the event completed */
int sntrup_event_query(void *ev);             /* SNTRUP_OK when complete, 1 when not yet */
void sntrup_event_destroy(void *ev);

/* Batch key generation with options (opt may be NULL = defaults). */
int sntrup_batch_keygen_ex(int param_set, uint64_t n_keys, uint64_t seed,
                           uint8_t *pk_out, uint8_t *sk_out, const sntrup_keygen_opts *opt);

/* Exact device workspace bytes a keygen call of this shape takes (what it carves from the
   caller's workspace, or the minimum the cached per-stream workspace is grown to; the cache
   allocates this + 1/8 + 1 MiB of slack).  Host-output calls additionally hold a library-owned
   staging allocation.  0 for an unknown parameter set, n_keys == 0 or a bad batch size.
   The plain form assumes default options (flags 0, default chunking). */
size_t sntrup_keygen_workspace_bytes(int param_set, uint64_t n_keys, uint32_t batch_size);
size_t sntrup_keygen_workspace_bytes_ex(int param_set, uint64_t n_keys, uint32_t batch_size,
                                        uint32_t flags, uint64_t chunk_keys);
/* Introspection (tests): bytes currently allocated for `stream` on the current device --
   which = 0: the cached workspace, 1: the host-output staging; 0 if none. */
size_t sntrup_workspace_reserved_bytes(void *stream, int which);

/* c[i] = a[i] * b[i] in R/q for i < n (the ring product of P:5339-5442: full product, then
   reduction by x^p - x - 1, coefficients centered).  a, b, c: int16 [n][p8], no aliasing of c
   with a or b.  Stream-ordered; returns after enqueueing. */
int rq_mul_batch(int param_set, uint64_t n, const int16_t *a, const int16_t *b, int16_t *c,
                 void *stream);

/* Big x small product (the paper's dedicated "big x small" R/q multiplier, P:6856-6866,
   P:6984-7104): c[i] = a[i] * b[i] in R/q with a int16 [n][p8] centered and b int8 [n][p16]
   with |b_j| <= 127 (ternary in the method: g, f, 3f); c int16 [n][p8].  Stream-ordered. */
int rq_mul_small_batch(int param_set, uint64_t n, const int16_t *a, const int8_t *b, int16_t *c,
                       void *stream);

/* c[i] = a[i] * b[i] in R/3: int8 [n][p16] rows in {-1,0,1}.  Stream-ordered. */
int r3_mul_batch(int param_set, uint64_t n, const int8_t *a, const int8_t *b, int8_t *c,
                 void *stream);

/* ---- Full-size secret key (reading Z24).  The paper's
   key-pair storage is 2512 / 2921 / 3321 bytes (App. D) = pk + an sk
   of 3 ceil(p/4) + |pk| + 32 bytes; it names neither the extra secret nor the hash.  Ours:
   sk_full = sk || pk || rho || SHA-512(0x04 || pk)[0..32), rho = ceil(p/4) bytes of stream
   domain 2^63 of the key (C2). */

/* Bytes of one full sk row (1763 for 761); 0 for an unknown parameter set. */
size_t sntrup_full_sk_bytes(int param_set);

/* sk_full[i] for global key indices first_key_index + i from that key's pk and sk rows.  All
   pointers DEVICE: pk u8 [n][pk_bytes], sk u8 [n][sk_bytes] (as sntrup_batch_keygen writes
   them), sk_full u8 [n][sntrup_full_sk_bytes].  Stream-ordered; SNTRUP_E_PARAM / SNTRUP_E_ARG
   (n == 0 or a NULL pointer) / SNTRUP_E_CUDA. */
int sntrup_full_sk_batch(int param_set, uint64_t n, uint64_t seed, uint64_t first_key_index,
                         const uint8_t *pk, const uint8_t *sk, uint8_t *sk_full, void *stream);

/* ---- Encapsulation / decapsulation core.  The paper benchmarks
   enc/dec (Table 1) for keys of shape (h, (f, 1/g)) but does not spell
   them out; the core follows Streamlined NTRU Prime as SPEC.md's encrypt_core/decrypt_core
   (S:405-422).  Hashing / ciphertext encoding (the KEM wrapper) are out of scope. */

/* r_out[i] = Short element (weight w) from stream domain `domain` of global key index
   first_key_index + i (C2-C4; domains >= 2^32 are reserved for encapsulation).
   int8 [n][p16].  Stream-ordered. */
int sntrup_sample_short_batch(int param_set, uint64_t n, uint64_t seed, uint64_t first_key_index,
                              uint64_t domain, int8_t *r_out, void *stream);

/* a_out[i] = uniform R/q element of SURVEY.md 8(c) C12 (the R/q microbenchmark's operand,
   BASELINE configs[2]) from stream domain `domain` of global key index first_key_index + i:
   a_j = floor(u_j q / 2^32) - (q-1)/2 with u the domain's 32-bit words (C2).
   int16 [n][p8] device, pad 0.  Stream-ordered; SNTRUP_E_PARAM / SNTRUP_E_ARG (n == 0, NULL). */
int sntrup_sample_uniform_rq_batch(int param_set, uint64_t n, uint64_t seed, uint64_t first_key_index,
                                   uint64_t domain, int16_t *a_out, void *stream);

/* c[i] = Round(h[i] * r[i]) in R/q: each centered coefficient to the nearest multiple of 3.
   h, c int16 [n][p8] centered; r int8 [n][p16] (weight w).  Stream-ordered. */
int sntrup_encap_core_batch(int param_set, uint64_t n, const int16_t *h, const int8_t *r, int16_t *c,
                            void *stream);

/* r_out[i] = ((3 f[i] * c[i] in R/q) mod 3) * ginv[i] in R/3, ok[i] = (weight(r_out[i]) == w).
   f, ginv, r_out int8 [n][p16]; c int16 [n][p8]; ok uint8 [n].  Uses the stream's workspace.
   Stream-ordered. */
int sntrup_decap_core_batch(int param_set, uint64_t n, const int8_t *f, const int8_t *ginv,
                            const int16_t *c, int8_t *r_out, uint8_t *ok, void *stream);

/* out[i] = 1/a[i] in R/q (batchInv) using product trees of batch_size leaves
   (0 -> 32), one constant-time divstep inversion per tree.  a, out: int16 [n][p8].
   If some a[i] == 0: returns SNTRUP_E_NOT_INVERTIBLE, *bad_index (host pointer, may be NULL)
   = the smallest such i, and out is unspecified.  Synchronous. */
int rq_recip_batch(int param_set, uint64_t n, const int16_t *a, int16_t *out,
                   uint32_t batch_size, uint64_t *bad_index, void *stream);

/* out[i] = 1/g[i] in R/3 for invertible g[i] (ok[i] = 1); non-invertible g[i] (ok[i] = 0,
   out[i] = 0).  Non-invertibility is a normal outcome, not an error.  g, out: int8 [n][p16];
   ok: uint8 [n] (device).  Synchronous. */
int r3_recip_batch(int param_set, uint64_t n, const int8_t *g, int8_t *out, uint8_t *ok,
                   uint32_t batch_size, void *stream);

/* isInvertible for n elements of R/3: ok[i] = 1 iff g[i] is a unit.
   Synchronous. */
int r3_is_invertible_batch(int param_set, uint64_t n, const int8_t *g, uint8_t *ok, void *stream);

/* pk[i] = Rq-encode(h[i]) (radix encoding, C10): h int16 [n][p8] -> uint8 [n][pk_bytes].
   Stream-ordered. */
int rq_encode_batch(int param_set, uint64_t n, const int16_t *h, uint8_t *pk, void *stream);

/* ---- Key pool: the paper's engNTRU batch_lib provider (section 4.2) on the GPU.
   A pinned host ring of `capacity` key pairs (a multiple of batch_keys, at least two batches),
   filled by sntrup_batch_keygen_ex calls of batch_keys keys (product trees of batch_size, 0 ->
   32) on a private stream, with consecutive global key indices first_key_index, +1, ... of
   `seed`.  The first take() fills lazily and waits; every take() that leaves the ring at most
   half full starts the next batch asynchronously, so a steady consumer does not wait for the GPU
   (the paper's "first key 2.5 ms, then 0 ms").  Thread-safe; one pool per device
   and parameter set as the caller chooses.  Handed-out slots are erased. */
typedef struct sntrup_pool sntrup_pool;
int sntrup_pool_create(int param_set, uint64_t seed, uint64_t first_key_index, uint64_t capacity,
                       uint64_t batch_keys, uint32_t batch_size, sntrup_pool **out);
/* Next key pair into HOST buffers pk (pk_bytes) and sk (sk_bytes); *key_index (may be NULL) =
   its global key index.  Blocks only if no generated key is left. */
int sntrup_pool_take(sntrup_pool *pool, uint8_t *pk, uint8_t *sk, uint64_t *key_index);
/* Counters: keys handed out, keys generated (incl. in flight), takes that had to wait for the
   GPU, keys ready or in flight.  Any pointer may be NULL. */
int sntrup_pool_stats(sntrup_pool *pool, uint64_t *taken, uint64_t *generated, uint64_t *waits,
                      uint64_t *ready);
void sntrup_pool_destroy(sntrup_pool *pool);

/* Release the cached device workspaces and host-output staging (all streams). */
void sntrup_release_workspace(void);
/* Synchronise `stream`, erase (zero) and free its cached workspace and staging (they hold secret
   f, 1/g and tree rows).  SNTRUP_OK or SNTRUP_E_CUDA. */
int sntrup_release_stream_workspace(void *stream);

/* Measurement hook: n ring products at p' = 383 --
   one sub-product of a one-level Karatsuba split of a 761 product -- through the same tensor-core
   kernels as the 761 products.  kind 0: R/3 (int8 rows of 384, fp4 MMAs); kind 1: R/q big x big
   mod 4591 (int16 rows of 384, int8 2 x 2 limbs); kinds 2 / 3: R/3 at p' = 255 / 257 (int8 rows
   of 256 / 272), the sub-product sizes of the paper's 5-way R/3 multiplier.  Device
   pointers; stream-ordered.  SNTRUP_OK / SNTRUP_E_ARG. */
int sntrup_probe_half_mul(int kind, uint64_t n, const void *a, const void *b, void *c, void *stream);

/* Integer-pipe peak (measurement for bench.py's roofline; BASELINE metric "int-pipe % of peak"):
   op 0 = IMAD (FMA pipe), 1 = IADD3, 2 = LOP3, 3 = SHF (ALU pipe).  A full-occupancy kernel of 8
   independent chains per thread of that one instruction; *lane_ops_per_clk_sm = lane-ops per SM
   clock per SM (from in-kernel clock64 spans per SM, clock-independent), *lane_ops_per_s = the
   whole GPU's lane-ops/s at the clock of this run (CUDA events).  Synchronous; device 0-stream. */
int sntrup_measure_int_peak(int op, double *lane_ops_per_clk_sm, double *lane_ops_per_s);

/* Role timing of the warp-specialised ring-product kernels: only in a build with
   -DSNTRUP_WS_TRACE (scripts/ws_trace.py); returns the number of counters (160 SM slots x 16
   roles' summed cycles) or 0 in a normal build.  The first call allocates the buffer. */
int sntrup_ws_trace_read(int reset, uint64_t *out, int n);

/* Number of kernels this library launched since load (device work only; for bench accounting). */
uint64_t sntrup_kernel_launch_count(void);

/* Select the ring-product implementation used by every call (measurement / A-B evidence):
   0 = tensor cores (the default): tcgen05.mma kind::mxf4 (e2m1) for small x small products
       (R/3, 3f x 3f), kind::i8 (int8 limbs) otherwise; in the down-sweeps the two children
       of a parent share one A operand;
   1 = int32 schoolbook on the integer pipes (v1);
   2 = int8 tensor cores only, one product per work item (v2);
   3 = int8 tensor cores only, with the shared-A R/3 down-sweep;
   4 = as 0, plus big x small products on fp4 with balanced base-9 digits (A/B only);
   5 = as 0, with the int8 products at MMA M = 64 instead of 128 (A/B only);
   6 = as 0, with one int8 big x big product per work item (A/B only);
   7 = as 0, with keygen's u_{2j} = g_{2j} * 3f_{2j+1} fused with the R/q tree's first level
       3f_{2j} * 3f_{2j+1} (shared A operand) instead of running on their own stream (A/B only);
   8 = as 0, with the int8 big x big products software-pipelined inside one CTA of 8 warps
       (two operand stages: item k+1 built and issued before item k's epilogue);
   9 = as 0, with the first K steps of the fp4 products' Hankel A operand written to TMEM
       (tcgen05.st) and read by the MMAs from there instead of from shared memory (128-column
       TMEM allocation per CTA); 10 = as 9 with 64 columns (fewer K steps in TMEM, more CTAs);
   11 = as 0, with the small x small (fp4) products on the warp-specialised persistent kernel
       whose Hankel A operand is built in registers and written to TMEM (csrc/tc4w.cuh);
   12 = as 0, with every K step of the fp4 products' A operand streamed through a 64-column TMEM
       window in rounds (no shared-memory A at all; 8 CTAs per SM);
   13 = as 0, with the int8 one-product items (R/q up-sweep, rq_mul_batch, rq_mul_small_batch) in
       the transposed Hankel form (csrc/tcxmul.cuh): 16 output coefficients per accumulator row,
       the folded operand read by the MMAs as a view of its staging array at MMA M = 64;
   14 = as 0, with the int8 big x big two-product items (R/q down-sweep, h) built and multiplied over
       the whole K range at once (72 KB of shared memory per CTA at p = 761, 3 CTAs per SM) instead of
       in two parts through half-size operand buffers (the default: 43 KB, 5 CTAs per SM);
   15 = as 0 with three parts; 16 = as 0 with the one-product int8 big x big items in two parts too.
   All are exact.  Variants 2-10 and 12-16 are compiled for sntrup761 only (other sets run 0, or 1 / 11);
   KEM pre/post-op calls always use the default kernel of their shape.  Returns SNTRUP_OK or
   SNTRUP_E_ARG. */
int sntrup_set_mul_impl(int impl);

/* A/B knob (measurement): threads per CTA of the R/q root inversion (one CTA per root, used when
   the roots are few): 128, 256 (default), 512 or 768; sntrup761 only.  SNTRUP_OK / SNTRUP_E_ARG. */
int sntrup_set_divstep_threads(int nt);

/* Knob: the root inversions used when the roots are few (fewer than two per SM).  0 (default) =
   automatic: jump-divsteps (App. D "jump-div-step"; csrc/jump.cuh: 31-step
   transition matrices decided by one warp on a 32-coefficient window, applied to (f, g) by the
   rest of that CTA and to (v, r) by the second CTA of a 2-CTA cluster) for the standalone
   reciprocal calls (rq_recip_batch, r3_recip_batch, r3_is_invertible_batch) and keygen calls of
   at most 4096 keys, whose time is the roots' latency; one divstep at a time inside larger keygen
   calls, where the roots overlap the other ring's products and the smaller SM footprint wins.  1 = one divstep at a time everywhere (R/q: 8 warps
   per root, one CTA barrier per step, sntrup_set_divstep_threads; R/3: one bitsliced warp per
   root); 2 = jump-divsteps everywhere.  + 4 (with 0 or 2): the jump CTAs reserve only the shared
   memory they use instead of more than half an SM each (measurement).  All variants are
   constant-time and exact.  Returns SNTRUP_OK or SNTRUP_E_ARG. */
int sntrup_set_root_impl(int impl);

/* Knob: scheduling of the tree tops inside bulk keygen calls (more than 4096 keys, ring streams).
   The top levels of the product trees (Algorithm 1 lines 10-11: batchInv) and the root
   inversions are chains of small launches; on their lane's stream they wait behind the other lane's
   bulk ring-product kernels, whose persistent CTAs hold the SMs' shared memory until the launch
   ends.  top_items > 0: ring-product launches of at most top_items products and the root
   inversions run on a high-priority companion stream of their chain (ordered with it by an event
   at each switch).  items_cap > 0: a ring-product launch uses at least ceil(work items /
   items_cap) CTAs, so a CTA retires after items_cap work items and a waiting high-priority CTA
   takes its place.  (0, 0) = off.  Outputs do not depend on it.  Returns SNTRUP_OK or
   SNTRUP_E_ARG (negative values). */
int sntrup_set_sched(long long top_items, long long items_cap);

/* Measurement hooks (bench.py).  When enabled, every kernel launch is bracketed by CUDA events
   recorded on its launching stream.  sntrup_profile_read() waits for the recorded events and
   returns, per kernel class, the summed device milliseconds, the summed work units, the summed
   algorithmic integer ops (ring products: 2 p^2 per product, the method's multiply-adds; 0 for
   other classes) and the launch count (classes:
   0 sample [keys], 1 R/3 product [products], 2 R/q product [products], 3 root inversions
   [inversions: R/3 roots, and in keygen both rings' roots in one launch], 4 R/q root inversion
   [inversions, rq_recip_batch], 5 repair [keys], 6 encode [keys], 7 other).
   Any output pointer may be NULL.  Returns the number of classes. */
void sntrup_profile_enable(int on);
/* Ring-product launches by arithmetic kind (0 = int8 tensor, 1 = fp4 tensor, 2 = int32
   schoolbook): summed device ms, algorithmic ops (2 p^2 per product) and launch counts since the
   last reset.  Returns the number of kinds (3). */
int sntrup_profile_read_kinds(int reset, double *ms, double *ops, uint64_t *launches);
/* As above, plus per kind the ring products computed and the bytes the tensor cores' MMAs fetched
   from shared memory (A and B tiles: work items x MMAs per item x tile bytes, from the kernels'
   geometry).  Algorithmic ops are 2 p^2 per ring product (the method's work), never per limb. */
int sntrup_profile_read_kinds_ex(int reset, double *ms, double *ops, uint64_t *launches, double *products,
                                 double *smem_bytes);
int sntrup_profile_read(int reset, double *ms, double *units, double *ops, uint64_t *launches,
                        int max_classes);

#ifdef __cplusplus
}
#endif
#endif /* SNTRUP_GPU_H */
