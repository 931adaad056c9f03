/*
 * sntrup_oracle.c -- plain, slow, obviously-correct CPU oracle for sntrup batch key generation.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference legs may load or call this library.  The product path
 * (paper_2106_08759_b200/, libsntrup_gpu.so) never links, imports or executes it, and this file
 * shares no code, header, table or constant generator with it.
 *
 * Citations: "P:N" = line N of PAPER.md (arXiv 2106.08759 LaTeX source); "C<k>" = the reading in
 * DESIGN.md §3 (taken from SURVEY.md §8(c)).  Everything here is exact integer arithmetic, one key
 * at a time, no batching, no blocking, no fusion:
 *   - ring product: schoolbook convolution, then fold with x^p = x + 1 ("reduce by
 *     x^p-x-1"), then centered reduction (D4)
 *   - inversion: textbook extended Euclid over GF(m)[x] (P:3539-3567 names ext-GCD inversion;
 *     the constant-time divstep variant is the GPU's business, not the oracle's)
 *   - KeyGen: P:3398-3461 (steps 1-5), one key per call; batching (Alg. 1) cannot
 *     change any output (C0: all results are unique), so the oracle does not batch.
 *
 * Parity status: every function below is pinned by tests/test_oracle_*.py against facts that
 * do not come from this file.  pk/sk byte formats are our own
 * conventions (C10/C11); compatibility with official sntrup761 KATs is "parity unpinned".
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <pthread.h>

/* ------------------------------------------------------------------------------------------ */
/* C2: SplitMix64, counter form.  SM(s, j) = output j (0-based) of SplitMix64 started at s.    */
/* ------------------------------------------------------------------------------------------ */
static uint64_t mix64(uint64_t z)
{
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}

uint64_t or_sm(uint64_t s, uint64_t j)
{
    return mix64(s + (j + 1) * 0x9E3779B97F4A7C15ULL);
}

/* 32-bit words u_0..u_{n-1} of domain d of key k: K = SM(seed,k); D = SM(K,d);
   u_{2j} = low32(SM(D,j)), u_{2j+1} = high32(SM(D,j)). */
void or_stream_words(uint64_t seed, uint64_t k, uint64_t d, int n, uint32_t *u)
{
    uint64_t K = or_sm(seed, k);
    uint64_t D = or_sm(K, d);
    for (int i = 0; i < n; i++) {
        uint64_t z = or_sm(D, (uint64_t)(i / 2));
        u[i] = (i % 2 == 0) ? (uint32_t)(z & 0xFFFFFFFFULL) : (uint32_t)(z >> 32);
    }
}

/* C3: Small: g_i = floor(3 * (u_i mod 2^30) / 2^30) - 1 */
void or_small_from_words(int p, const uint32_t *u, int8_t *g)
{
    for (int i = 0; i < p; i++) {
        uint64_t t = (uint64_t)(u[i] & 0x3FFFFFFFu);
        g[i] = (int8_t)((int)((3 * t) >> 30) - 1);
    }
}

/* C4: Short (fixed weight w) by sorting p tagged 32-bit draws. */
static int cmp_u32(const void *x, const void *y)
{
    uint32_t a = *(const uint32_t *)x, b = *(const uint32_t *)y;
    return (a > b) - (a < b);
}

void or_short_from_words(int p, int w, const uint32_t *u, int8_t *f)
{
    uint32_t *L = (uint32_t *)malloc(sizeof(uint32_t) * (size_t)p);
    for (int i = 0; i < p; i++) {
        if (i < w) L[i] = u[i] & 0xFFFFFFFEu;            /* low bits 00 or 10 -> -1 / +1 */
        else       L[i] = (u[i] & 0xFFFFFFFCu) | 1u;     /* low bits 01       ->  0      */
    }
    qsort(L, (size_t)p, sizeof(uint32_t), cmp_u32);
    for (int i = 0; i < p; i++) f[i] = (int8_t)((int)(L[i] & 3u) - 1);
    free(L);
}

/* C12: uniform R/q element of the R/q microbenchmark (BASELINE configs[2]):
   a_j = floor(u_j * q / 2^32) - (q-1)/2, j = 0..p-1, from the words of its stream domain. */
void or_uniform_from_words(int p, int q, const uint32_t *u, int16_t *a)
{
    for (int j = 0; j < p; j++) {
        uint64_t t = ((uint64_t)u[j] * (uint64_t)q) >> 32;
        a[j] = (int16_t)((int64_t)t - (q - 1) / 2);
    }
}

/* ------------------------------------------------------------------------------------------ */
/* Arithmetic in Z/m and (Z/m)[x]                                                               */
/* ------------------------------------------------------------------------------------------ */
static int64_t mod_pos(int64_t a, int64_t m)     /* representative in [0, m) */
{
    int64_t r = a % m;
    return r < 0 ? r + m : r;
}

static int64_t mod_center(int64_t a, int64_t m)  /* representative in [-(m-1)/2, (m-1)/2] (m odd) */
{
    int64_t r = mod_pos(a, m);
    return r > (m - 1) / 2 ? r - m : r;
}

static int64_t inv_scalar(int64_t a, int64_t m)  /* 1/a mod m via integer extended Euclid; a != 0 */
{
    int64_t r0 = m, r1 = mod_pos(a, m), s0 = 0, s1 = 1;
    while (r1 != 0) {
        int64_t qq = r0 / r1, t;
        t = r0 - qq * r1; r0 = r1; r1 = t;
        t = s0 - qq * s1; s0 = s1; s1 = t;
    }
    /* r0 == gcd == 1 for prime m */
    return mod_pos(s0, m);
}

/* C7: c = a*b in (Z/m)[x]/(x^p - x - 1).
   1. schoolbook c_k = sum_{i+j=k} a_i b_j, k = 0..2p-2, in int64;
   2. fold with x^p = x + 1: for k = 2p-2 down to p, c_{k-p} += c_k, c_{k-p+1} += c_k, c_k = 0;
   3. centered reduction mod m. */
void or_poly_mul(int p, int64_t m, const int64_t *a, const int64_t *b, int64_t *c)
{
    int64_t *t = (int64_t *)calloc((size_t)(2 * p - 1), sizeof(int64_t));
    for (int i = 0; i < p; i++)
        for (int j = 0; j < p; j++)
            t[i + j] += a[i] * b[j];
    for (int k = 2 * p - 2; k >= p; k--) {
        t[k - p] += t[k];
        t[k - p + 1] += t[k];
        t[k] = 0;
    }
    for (int k = 0; k < p; k++) c[k] = mod_center(t[k], m);
    free(t);
}

/* --- dense polynomials over GF(m) with explicit degree (deg -1 = zero polynomial) --- */
static int poly_deg(const int64_t *a, int n)
{
    for (int i = n - 1; i >= 0; i--) if (a[i] != 0) return i;
    return -1;
}

/* C5/C6: 1/a in (Z/m)[x]/(x^p-x-1) by the extended Euclidean algorithm on (F, a), F = x^p-x-1:
   r0 = F, r1 = a, s0 = 0, s1 = 1; while r1 != 0: (q, r) = divmod(r0, r1);
   (r0, r1) = (r1, r); (s0, s1) = (s1, s0 - q*s1).   Invariant s_i * a == r_i (mod F).
   a is invertible iff deg r0 == 0 at the end; then 1/a = s0 / r0[0] (reduced mod F).
   Returns 1 and writes the centered inverse if invertible, else returns 0 and writes zeros. */
int or_poly_inv(int p, int64_t m, const int64_t *a, int64_t *out)
{
    int n = p + 1;                                   /* room for degree <= p */
    int64_t *r0 = calloc((size_t)n, 8), *r1 = calloc((size_t)n, 8);
    int64_t *s0 = calloc((size_t)(2 * n), 8), *s1 = calloc((size_t)(2 * n), 8);
    int64_t *qt = calloc((size_t)n, 8), *tmp = calloc((size_t)(2 * n), 8);
    int ok = 0;

    r0[0] = mod_pos(-1, m); r0[1] = mod_pos(-1, m); r0[p] = 1;          /* F = x^p - x - 1 */
    for (int i = 0; i < p; i++) r1[i] = mod_pos(a[i], m);
    s1[0] = 1;

    while (poly_deg(r1, n) >= 0) {
        int d0 = poly_deg(r0, n), d1 = poly_deg(r1, n);
        /* long division r0 = qt*r1 + rem, rem left in r0 */
        memset(qt, 0, (size_t)n * 8);
        int64_t lead_inv = inv_scalar(r1[d1], m);
        for (int k = d0 - d1; k >= 0; k--) {
            int64_t coef = mod_pos(r0[k + d1] * lead_inv, m);
            qt[k] = coef;
            if (coef == 0) continue;
            for (int i = 0; i <= d1; i++)
                r0[k + i] = mod_pos(r0[k + i] - coef * r1[i], m);
        }
        /* (r0, r1) <- (r1, rem) */
        int64_t *sw = r0; r0 = r1; r1 = sw;
        /* (s0, s1) <- (s1, s0 - qt*s1) */
        memset(tmp, 0, (size_t)(2 * n) * 8);
        int dq = poly_deg(qt, n), ds = poly_deg(s1, 2 * n);
        for (int i = 0; i <= dq; i++)
            for (int j = 0; j <= ds; j++)
                tmp[i + j] = mod_pos(tmp[i + j] + qt[i] * s1[j], m);
        for (int i = 0; i < 2 * n; i++) tmp[i] = mod_pos(s0[i] - tmp[i], m);
        sw = s0; s0 = s1; s1 = tmp; tmp = sw;
    }

    if (poly_deg(r0, n) == 0) {
        ok = 1;
        int64_t c = inv_scalar(r0[0], m);
        /* reduce s0 mod F by folding (deg s0 < p holds for Euclid, fold kept for safety) */
        for (int k = 2 * n - 1; k >= p; k--) {
            if (s0[k] == 0) continue;
            s0[k - p] = mod_pos(s0[k - p] + s0[k], m);
            s0[k - p + 1] = mod_pos(s0[k - p + 1] + s0[k], m);
            s0[k] = 0;
        }
        for (int i = 0; i < p; i++) out[i] = mod_center(s0[i] * c, m);
    } else {
        for (int i = 0; i < p; i++) out[i] = 0;
    }
    free(r0); free(r1); free(s0); free(s1); free(qt); free(tmp);
    return ok;
}

/* ------------------------------------------------------------------------------------------ */
/* Encodings (C10, C11)                                                                        */
/* ------------------------------------------------------------------------------------------ */
/* C10: mixed-radix Encode(R, M), recursive pair merge with threshold 2^14. Returns bytes written. */
static size_t encode_rec(const uint32_t *R, const uint32_t *M, int n, uint8_t *out)
{
    if (n == 0) return 0;
    size_t len = 0;
    if (n == 1) {
        uint32_t r = R[0], m = M[0];
        while (m > 1) {
            out[len++] = (uint8_t)(r & 255u);
            r >>= 8;
            m = (m + 255u) >> 8;
        }
        return len;
    }
    int n2 = (n + 1) / 2;
    uint32_t *R2 = malloc(sizeof(uint32_t) * (size_t)n2), *M2 = malloc(sizeof(uint32_t) * (size_t)n2);
    for (int i = 0; i + 1 < n; i += 2) {
        uint32_t m = M[i] * M[i + 1];
        uint32_t r = R[i] + M[i] * R[i + 1];
        while (m >= 16384u) {
            out[len++] = (uint8_t)(r & 255u);
            r >>= 8;
            m = (m + 255u) >> 8;
        }
        R2[i / 2] = r; M2[i / 2] = m;
    }
    if (n & 1) { R2[n2 - 1] = R[n - 1]; M2[n2 - 1] = M[n - 1]; }
    len += encode_rec(R2, M2, n2, out + len);
    free(R2); free(M2);
    return len;
}

/* Decode: inverse of encode_rec.  Returns bytes consumed, or (size_t)-1 on a range violation. */
static size_t decode_rec(const uint8_t *S, const uint32_t *M, int n, uint32_t *R)
{
    if (n == 0) return 0;
    if (n == 1) {
        uint32_t m = M[0];
        uint64_t r = 0, scale = 1;
        size_t len = 0;
        while (m > 1) {
            r += (uint64_t)S[len++] * scale;
            scale <<= 8;
            m = (m + 255u) >> 8;
        }
        if (r >= M[0]) return (size_t)-1;
        R[0] = (uint32_t)r;
        return len;
    }
    int n2 = (n + 1) / 2;
    uint32_t *R2 = malloc(sizeof(uint32_t) * (size_t)n2), *M2 = malloc(sizeof(uint32_t) * (size_t)n2);
    int *emit = malloc(sizeof(int) * (size_t)n2);
    size_t here = 0;
    for (int i = 0; i + 1 < n; i += 2) {
        uint32_t m = M[i] * M[i + 1];
        int e = 0;
        while (m >= 16384u) { e++; m = (m + 255u) >> 8; }
        emit[i / 2] = e; M2[i / 2] = m; here += (size_t)e;
    }
    if (n & 1) { M2[n2 - 1] = M[n - 1]; emit[n2 - 1] = 0; }
    size_t sub = decode_rec(S + here, M2, n2, R2);
    if (sub == (size_t)-1) { free(R2); free(M2); free(emit); return (size_t)-1; }
    size_t pos = 0;
    for (int i = 0; i + 1 < n; i += 2) {
        int e = emit[i / 2];
        uint64_t r = R2[i / 2];
        for (int t = e - 1; t >= 0; t--) r = r * 256u + S[pos + (size_t)t];
        pos += (size_t)e;
        uint64_t lo = r % M[i], hi = r / M[i];
        if (hi >= M[i + 1]) { free(R2); free(M2); free(emit); return (size_t)-1; }
        R[i] = (uint32_t)lo; R[i + 1] = (uint32_t)hi;
    }
    if (n & 1) R[n - 1] = R2[n2 - 1];
    free(R2); free(M2); free(emit);
    return here + sub;
}

/* pk = Rq-encode(h): R_i = h_i + (q-1)/2, M_i = q. */
size_t or_rq_encode(int p, int q, const int16_t *h, uint8_t *out)
{
    uint32_t *R = malloc(sizeof(uint32_t) * (size_t)p), *M = malloc(sizeof(uint32_t) * (size_t)p);
    for (int i = 0; i < p; i++) { R[i] = (uint32_t)(h[i] + (q - 1) / 2); M[i] = (uint32_t)q; }
    size_t len = encode_rec(R, M, p, out);
    free(R); free(M);
    return len;
}

/* General Encode for tests (arbitrary R, M lists). */
size_t or_encode_general(int n, const uint32_t *R, const uint32_t *M, uint8_t *out)
{
    return encode_rec(R, M, n, out);
}

size_t or_decode_general(int n, const uint32_t *M, const uint8_t *S, uint32_t *R)
{
    return decode_rec(S, M, n, R);
}

/* Byte length of Rq-encode for (p, q): depends only on M (C10). */
size_t or_rq_encoded_bytes(int p, int q)
{
    uint32_t *R = calloc((size_t)p, sizeof(uint32_t)), *M = malloc(sizeof(uint32_t) * (size_t)p);
    uint8_t *buf = malloc((size_t)(4 * p + 16));
    for (int i = 0; i < p; i++) M[i] = (uint32_t)q;
    size_t len = encode_rec(R, M, p, buf);
    free(R); free(M); free(buf);
    return len;
}

int or_rq_decode(int p, int q, const uint8_t *in, int16_t *h)
{
    uint32_t *R = malloc(sizeof(uint32_t) * (size_t)p), *M = malloc(sizeof(uint32_t) * (size_t)p);
    for (int i = 0; i < p; i++) M[i] = (uint32_t)q;
    size_t len = decode_rec(in, M, p, R);
    if (len != (size_t)-1)
        for (int i = 0; i < p; i++) h[i] = (int16_t)((int)R[i] - (q - 1) / 2);
    free(R); free(M);
    return len == (size_t)-1 ? -1 : 0;
}

/* C11: Small-encode: byte_j = sum_{t=0..3} (c_{4j+t} + 1) * 4^t over present coefficients. */
void or_small_encode(int p, const int8_t *c, uint8_t *out)
{
    int nb = (p + 3) / 4;
    for (int j = 0; j < nb; j++) {
        int v = 0;
        for (int t = 0; t < 4; t++) {
            int i = 4 * j + t;
            if (i < p) v += (c[i] + 1) << (2 * t);
        }
        out[j] = (uint8_t)v;
    }
}

void or_small_decode(int p, const uint8_t *in, int8_t *c)
{
    for (int i = 0; i < p; i++) c[i] = (int8_t)((int)((in[i / 4] >> (2 * (i % 4))) & 3) - 1);
}

/* ------------------------------------------------------------------------------------------ */
/* KeyGen, one key, with the C2 domain-separated streams.                         */
/* ------------------------------------------------------------------------------------------ */
/* Returns 0 on success, -1 if no invertible g was found within max_attempts draws.
   Outputs (each optional, may be NULL): g, f, ginv (int8[p]), h (int16[p]), attempts,
   pk (or_rq_encoded_bytes), sk (2*ceil(p/4)). */
int or_keygen(int p, int q, int w, uint64_t seed, uint64_t k, int max_attempts,
              int8_t *g_out, int8_t *f_out, int8_t *ginv_out, int16_t *h_out, int *attempts_out,
              uint8_t *pk_out, uint8_t *sk_out)
{
    uint32_t *u = malloc(sizeof(uint32_t) * (size_t)p);
    int8_t *g = malloc((size_t)p), *f = malloc((size_t)p), *gi = malloc((size_t)p);
    int64_t *A = malloc(8 * (size_t)p), *B = malloc(8 * (size_t)p), *C = malloc(8 * (size_t)p);
    int16_t *h = malloc(2 * (size_t)p);
    int attempt, rc = 0;

    /* Step 1 (+ P:3414-3418 "repeat until g is invertible in R/3"): attempt a uses domain 1+a. */
    for (attempt = 0; attempt < max_attempts; attempt++) {
        or_stream_words(seed, k, 1 + (uint64_t)attempt, p, u);
        or_small_from_words(p, u, g);
        for (int i = 0; i < p; i++) A[i] = g[i];
        if (or_poly_inv(p, 3, A, B)) break;                  /* step 2: 1/g in R/3 */
    }
    if (attempt == max_attempts) { rc = -1; goto done; }
    for (int i = 0; i < p; i++) gi[i] = (int8_t)B[i];

    /* Step 3: f in Short from domain 0 (reading Z4: independent of the g attempts). */
    or_stream_words(seed, k, 0, p, u);
    or_short_from_words(p, w, u, f);

    /* Step 4: h = g / (3f) in R/q: u = 1/(3f) by Euclid, then h = g * u. */
    for (int i = 0; i < p; i++) A[i] = 3 * (int64_t)f[i];
    if (!or_poly_inv(p, q, A, B)) { rc = -2; goto done; }    /* impossible: R/q is a field */
    for (int i = 0; i < p; i++) A[i] = g[i];
    or_poly_mul(p, q, A, B, C);
    for (int i = 0; i < p; i++) h[i] = (int16_t)C[i];

    /* Step 5: output (h, (f, 1/g)), encoded per C10/C11. */
    if (g_out) memcpy(g_out, g, (size_t)p);
    if (f_out) memcpy(f_out, f, (size_t)p);
    if (ginv_out) memcpy(ginv_out, gi, (size_t)p);
    if (h_out) memcpy(h_out, h, 2 * (size_t)p);
    if (pk_out) or_rq_encode(p, q, h, pk_out);
    if (sk_out) {
        int nb = (p + 3) / 4;
        or_small_encode(p, f, sk_out);
        or_small_encode(p, gi, sk_out + nb);
    }
done:
    if (attempts_out) *attempts_out = attempt + 1;
    free(u); free(g); free(f); free(gi); free(A); free(B); free(C); free(h);
    return rc;
}

/* ------------------------------------------------------------------------------------------ */
/* Many keys: independent per-key calls spread over host threads (parallel over keys only).     */
/* ------------------------------------------------------------------------------------------ */
typedef struct {
    int p, q, w; uint64_t seed;
    const uint64_t *indices; uint64_t n;       /* global key indices to compute */
    uint8_t *pk; size_t pk_stride; uint8_t *sk; size_t sk_stride;
    int16_t *h; int8_t *g, *f, *ginv; size_t row; int32_t *attempts;
    uint64_t next; pthread_mutex_t mu; int err;
} many_job;

static void *many_worker(void *arg)
{
    many_job *J = (many_job *)arg;
    for (;;) {
        pthread_mutex_lock(&J->mu);
        uint64_t i = J->next++;
        pthread_mutex_unlock(&J->mu);
        if (i >= J->n) break;
        int att = 0;
        int rc = or_keygen(J->p, J->q, J->w, J->seed, J->indices[i], 255,
                           J->g ? J->g + i * J->row : NULL, J->f ? J->f + i * J->row : NULL,
                           J->ginv ? J->ginv + i * J->row : NULL, J->h ? J->h + i * J->row : NULL,
                           &att, J->pk ? J->pk + i * J->pk_stride : NULL,
                           J->sk ? J->sk + i * J->sk_stride : NULL);
        if (J->attempts) J->attempts[i] = att;
        if (rc) { pthread_mutex_lock(&J->mu); J->err = rc; pthread_mutex_unlock(&J->mu); }
    }
    return NULL;
}

/* Key i of the call is global key indices[i].  Rows of g/f/ginv/h have stride `row` elements. */
int or_keygen_many(int p, int q, int w, uint64_t seed, const uint64_t *indices, uint64_t n,
                   int n_threads, uint8_t *pk, size_t pk_stride, uint8_t *sk, size_t sk_stride,
                   int16_t *h, int8_t *g, int8_t *f, int8_t *ginv, size_t row, int32_t *attempts)
{
    many_job J = {p, q, w, seed, indices, n, pk, pk_stride, sk, sk_stride, h, g, f, ginv, row,
                  attempts, 0, PTHREAD_MUTEX_INITIALIZER, 0};
    if (n_threads < 1) n_threads = 1;
    pthread_t *th = malloc(sizeof(pthread_t) * (size_t)n_threads);
    for (int t = 0; t < n_threads; t++) pthread_create(&th[t], NULL, many_worker, &J);
    for (int t = 0; t < n_threads; t++) pthread_join(th[t], NULL);
    free(th);
    return J.err;
}

/* Batched ring products c[i] = a[i]*b[i] in R/q (int16 centered rows of stride `row`), threaded.
   Used for the rq_mul_batch parity tests and the cpu_baseline of the R/q microbenchmark. */
typedef struct {
    int p; int64_t m; const int16_t *a, *b; int16_t *c; size_t row; uint64_t n, next;
    pthread_mutex_t mu;
} mul_job;

static void *mul_worker(void *arg)
{
    mul_job *J = (mul_job *)arg;
    int64_t *A = malloc(8 * (size_t)J->p), *B = malloc(8 * (size_t)J->p), *C = malloc(8 * (size_t)J->p);
    for (;;) {
        pthread_mutex_lock(&J->mu);
        uint64_t i = J->next++;
        pthread_mutex_unlock(&J->mu);
        if (i >= J->n) break;
        for (int t = 0; t < J->p; t++) { A[t] = J->a[i * J->row + t]; B[t] = J->b[i * J->row + t]; }
        or_poly_mul(J->p, J->m, A, B, C);
        for (int t = 0; t < J->p; t++) J->c[i * J->row + t] = (int16_t)C[t];
    }
    free(A); free(B); free(C);
    return NULL;
}

void or_mul_many(int p, int64_t m, uint64_t n, const int16_t *a, const int16_t *b, int16_t *c,
                 size_t row, int n_threads)
{
    mul_job J = {p, m, a, b, c, row, n, 0, PTHREAD_MUTEX_INITIALIZER};
    if (n_threads < 1) n_threads = 1;
    pthread_t *th = malloc(sizeof(pthread_t) * (size_t)n_threads);
    for (int t = 0; t < n_threads; t++) pthread_create(&th[t], NULL, mul_worker, &J);
    for (int t = 0; t < n_threads; t++) pthread_join(th[t], NULL);
    free(th);
}

/* ------------------------------------------------------------------------------------------ */
/* Encapsulation / decapsulation core (SPEC.md encrypt_core /    */
/* decrypt_core, S:405-422 -- the paper only benchmarks enc/dec, Table 1, and names the */
/* key shape (h, (f, 1/g)) of section 3.1).  Plain definitions, one key at a time.  */
/*   encap: c = Round(h * r) in R/q, Round = each centered coefficient x to the nearest multiple   */
/*          of 3, x - (x mods 3) (unique: x is within 1 of exactly one multiple of 3; stays in   */
/*          range because (q-1)/2 = 0 mod 3 for every set, C1).                                 */
/*   decap: e = 3 f * c in R/q (centered); e3 = e mod 3 lifted to {-1,0,1}; r' = e3 * (1/g) in    */
/*          R/3; valid iff weight(r') = w.                                                        */
/* ------------------------------------------------------------------------------------------ */
void or_encap_core(int p, int q, const int16_t *h, const int8_t *r, int16_t *c)
{
    int64_t *H = calloc((size_t)p, sizeof(int64_t)), *R = calloc((size_t)p, sizeof(int64_t));
    int64_t *X = calloc((size_t)p, sizeof(int64_t));
    for (int i = 0; i < p; i++) { H[i] = h[i]; R[i] = r[i]; }
    or_poly_mul(p, q, H, R, X);
    for (int i = 0; i < p; i++) {
        const int64_t x = X[i];                     /* centered in [-(q-1)/2, (q-1)/2] */
        const int64_t m3 = mod_center(x, 3);        /* x - m3 is the nearest multiple of 3 */
        c[i] = (int16_t)(x - m3);
    }
    free(H); free(R); free(X);
}

int or_decap_core(int p, int q, int w, const int8_t *f, const int8_t *ginv, const int16_t *c,
                  int8_t *r_out)
{
    int64_t *F3 = calloc((size_t)p, sizeof(int64_t)), *C = calloc((size_t)p, sizeof(int64_t));
    int64_t *E = calloc((size_t)p, sizeof(int64_t)), *G = calloc((size_t)p, sizeof(int64_t));
    int64_t *R = calloc((size_t)p, sizeof(int64_t));
    for (int i = 0; i < p; i++) { F3[i] = 3 * (int64_t)f[i]; C[i] = c[i]; G[i] = ginv[i]; }
    or_poly_mul(p, q, F3, C, E);                    /* e = 3f * c in R/q, centered */
    for (int i = 0; i < p; i++) E[i] = mod_center(E[i], 3);
    or_poly_mul(p, 3, E, G, R);                     /* r' = e3 * (1/g) in R/3 */
    int weight = 0;
    for (int i = 0; i < p; i++) { r_out[i] = (int8_t)R[i]; weight += R[i] != 0; }
    free(F3); free(C); free(E); free(G); free(R);
    return weight == w;
}

/* ------------------------------------------------------------------------------------------ */
/* Full-size secret key (reading Z24 in DESIGN.md): the paper stores key    */
/* pairs of 2512 / 2921 / 3321 bytes (App. D) = pk + an sk of         */
/* 3 ceil(p/4) + |pk| + 32 bytes, but names neither the extra secret rho nor the hash.  Ours:     */
/*   sk_full = Small(f) || Small(1/g) || pk || rho || H(pk)                                     */
/*   rho     = ceil(p/4) bytes of key k's stream domain OR_DOMAIN_RHO (C2), little-endian words  */
/*   H(pk)   = SHA-512(0x04 || pk)[0..32)  (FIPS 180-4, written out below, one block at a time)  */
/* ------------------------------------------------------------------------------------------ */
#include "sha512_consts.h"

#define OR_DOMAIN_RHO 0x8000000000000000ULL

static uint64_t rotr64(uint64_t x, int n) { return (x >> n) | (x << (64 - n)); }

/* FIPS 180-4 6.4.2: one 1024-bit block into the hash state */
static void sha512_block(uint64_t H[8], const uint8_t blk[128])
{
    uint64_t W[80];
    for (int t = 0; t < 16; t++) {
        uint64_t w = 0;
        for (int b = 0; b < 8; b++) w = (w << 8) | blk[8 * t + b];     /* big-endian words */
        W[t] = w;
    }
    for (int t = 16; t < 80; t++) {
        const uint64_t s0 = rotr64(W[t - 15], 1) ^ rotr64(W[t - 15], 8) ^ (W[t - 15] >> 7);
        const uint64_t s1 = rotr64(W[t - 2], 19) ^ rotr64(W[t - 2], 61) ^ (W[t - 2] >> 6);
        W[t] = s1 + W[t - 7] + s0 + W[t - 16];
    }
    uint64_t a = H[0], b = H[1], c = H[2], d = H[3], e = H[4], f = H[5], g = H[6], h = H[7];
    for (int t = 0; t < 80; t++) {
        const uint64_t S1 = rotr64(e, 14) ^ rotr64(e, 18) ^ rotr64(e, 41);
        const uint64_t ch = (e & f) ^ (~e & g);
        const uint64_t T1 = h + S1 + ch + OR_SHA512_K[t] + W[t];
        const uint64_t S0 = rotr64(a, 28) ^ rotr64(a, 34) ^ rotr64(a, 39);
        const uint64_t maj = (a & b) ^ (a & c) ^ (b & c);
        const uint64_t T2 = S0 + maj;
        h = g; g = f; f = e; e = d + T1; d = c; c = b; b = a; a = T1 + T2;
    }
    H[0] += a; H[1] += b; H[2] += c; H[3] += d; H[4] += e; H[5] += f; H[6] += g; H[7] += h;
}

/* SHA-512 of msg[0..len) (FIPS 180-4 5.1.2 padding: 0x80, zeros, 128-bit big-endian bit length) */
void or_sha512(const uint8_t *msg, size_t len, uint8_t out[64])
{
    uint64_t H[8];
    for (int i = 0; i < 8; i++) H[i] = OR_SHA512_H0[i];
    const size_t total = ((len + 17 + 127) / 128) * 128;
    uint8_t *buf = calloc(total, 1);
    memcpy(buf, msg, len);
    buf[len] = 0x80;
    const uint64_t bits = (uint64_t)len * 8;
    for (int b = 0; b < 8; b++) buf[total - 1 - b] = (uint8_t)(bits >> (8 * b));
    for (size_t o = 0; o < total; o += 128) sha512_block(H, buf + o);
    free(buf);
    for (int i = 0; i < 8; i++)
        for (int b = 0; b < 8; b++) out[8 * i + b] = (uint8_t)(H[i] >> (56 - 8 * b));
}

/* full sk of global key index k from its pk and sk bytes; returns the bytes written */
size_t or_full_sk(int p, uint64_t seed, uint64_t k, const uint8_t *pk, size_t pkb,
                  const uint8_t *sk, size_t skb, uint8_t *out)
{
    const size_t rb = (size_t)((p + 3) / 4);
    size_t o = 0;
    memcpy(out + o, sk, skb); o += skb;
    memcpy(out + o, pk, pkb); o += pkb;
    const uint64_t D = or_sm(or_sm(seed, k), OR_DOMAIN_RHO);
    for (size_t j = 0; j < rb; j++) out[o + j] = (uint8_t)(or_sm(D, j / 8) >> (8 * (j % 8)));
    o += rb;
    uint8_t *m = malloc(pkb + 1);
    m[0] = 4;
    memcpy(m + 1, pk, pkb);
    uint8_t hsh[64];
    or_sha512(m, pkb + 1, hsh);
    free(m);
    memcpy(out + o, hsh, 32);
    o += 32;
    return o;
}
