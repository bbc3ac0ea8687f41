/* sj_oracle.c -- CPU restatement of the reference's join arithmetic.
 *
 * TEST INFRASTRUCTURE ONLY.  Nothing in paper_2312_01476_b200/ links or calls
 * this file; only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline
 * leg use it, and only as the checker.
 *
 * Every function restates one reference routine (paths relative to
 * /root/reference/pkg/src/simjoin/):
 *
 *   oc_fnv1a64          <- sj_fnv1a64            _kernelcore.c:33-40
 *   oc_synthetic_fill   <- splitmix64 + sj_synthetic_fill  _kernelcore.c:42-50, 72-80
 *   oc_normalize_rows   <- normalize_row + sj_normalize_rows _kernelcore.c:52-70, 82-87
 *   oc_row_norms        <- sj_row_norms           _kernelcore.c:89-99
 *   oc_dot_seq          <- sj_dot_seq + MADD      _kernelcore.c:21-25, 101-106
 *                          (x86 FMA build: one fmaf per component, sequential in d)
 *   oc_join_count/fill  <- tensor_join semantics  join.py:317-373 (tile_dot cell ==
 *                          sj_dot_seq, scan `>= theta`, canonical (l, r) order
 *                          core.py:196-213).  Brute force, row-major, so the
 *                          emitted order is already canonical.
 *   oc_subword_embed    <- NOT in the reference (SPEC.md:175 lists subword hashing
 *                          as a non-goal).  Builder-pinned restatement of the cfg3
 *                          FastText-style model; see DESIGN.md "subword model".
 *
 * Build: oracle/Makefile (gcc -O2 -ffp-contract=off).  fmaf() is the libm
 * correctly-rounded fused multiply-add, so the canonical value does not
 * depend on whether this host has hardware FMA.
 */
#include <math.h>
#include <stdint.h>
#include <string.h>

uint64_t oc_fnv1a64(const uint8_t* data, int64_t n) {
    uint64_t h = 0xcbf29ce484222325ULL;
    for (int64_t i = 0; i < n; i++) {
        h ^= (uint64_t)data[i];
        h *= 0x100000001b3ULL;
    }
    return h;
}

/* Batched: tokens packed in `bytes`, token t = bytes[offs[t], offs[t+1]). */
void oc_fnv1a64_many(const uint8_t* bytes, const int64_t* offs, int64_t n,
                     uint64_t xor_seed, uint64_t* out) {
    for (int64_t t = 0; t < n; t++)
        out[t] = oc_fnv1a64(bytes + offs[t], offs[t + 1] - offs[t]) ^ xor_seed;
}

static int oc_normalize_row(float* row, int64_t dim) {
    if (dim == 0) return 0;
    double ss = 0.0;
    for (int64_t d = 0; d < dim; d++) {
        double x = (double)row[d];
        double sq = x * x;            /* exact: 24-bit * 24-bit fits in 53 bits */
        ss = ss + sq;
    }
    double norm = sqrt(ss);
    int repaired = 0;
    if (norm < 1e-12) {
        row[0] = 1.0f;
        ss = 0.0;
        for (int64_t d = 0; d < dim; d++) {
            double x = (double)row[d];
            ss = ss + x * x;
        }
        norm = sqrt(ss);
        repaired = 1;
    }
    for (int64_t d = 0; d < dim; d++)
        row[d] = (float)((double)row[d] / norm);
    return repaired;
}

int64_t oc_normalize_rows(float* m, int64_t n, int64_t dim) {
    int64_t rep = 0;
    for (int64_t i = 0; i < n; i++) rep += oc_normalize_row(m + i * dim, dim);
    return rep;
}

void oc_row_norms(const float* m, int64_t n, int64_t dim, float* out) {
    for (int64_t i = 0; i < n; i++) {
        double ss = 0.0;
        for (int64_t d = 0; d < dim; d++) {
            double x = (double)m[i * dim + d];
            ss = ss + x * x;
        }
        out[i] = (float)sqrt(ss);
    }
}

void oc_synthetic_fill(uint64_t stream_seed, int64_t dim, float* out) {
    uint64_t state = stream_seed;
    for (int64_t d = 0; d < dim; d++) {
        state += 0x9E3779B97F4A7C15ULL;
        uint64_t z = state;
        z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
        z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
        z = z ^ (z >> 31);
        double v = ((double)z * 0x1p-64) * 2.0 - 1.0;
        out[d] = (float)v;
    }
    oc_normalize_row(out, dim);
}

void oc_synthetic_fill_many(const uint64_t* seeds, int64_t n, int64_t dim,
                            float* out) {
    for (int64_t i = 0; i < n; i++) oc_synthetic_fill(seeds[i], dim, out + i * dim);
}

float oc_dot_seq(const float* a, const float* b, int64_t dim) {
    float acc = 0.0f;
    for (int64_t d = 0; d < dim; d++) acc = fmaf(a[d], b[d], acc);
    return acc;
}

void oc_dots_vm(const float* a, const float* m, int64_t n, int64_t dim,
                float* out) {
    for (int64_t i = 0; i < n; i++) out[i] = oc_dot_seq(a, m + i * dim, dim);
}

/* Brute-force threshold join over normalized rows.  Rows [i0, i1) of L. */
int64_t oc_join_count(const float* L, int64_t i0, int64_t i1, const float* S,
                      int64_t ns, int64_t dim, float theta) {
    int64_t k = 0;
    for (int64_t i = i0; i < i1; i++)
        for (int64_t j = 0; j < ns; j++)
            if (oc_dot_seq(L + i * dim, S + j * dim, dim) >= theta) k++;
    return k;
}

int64_t oc_join_fill(const float* L, int64_t i0, int64_t i1, const float* S,
                     int64_t ns, int64_t dim, float theta, uint64_t* lefts,
                     uint64_t* rights, float* sims, int64_t cap) {
    int64_t k = 0;
    for (int64_t i = i0; i < i1; i++)
        for (int64_t j = 0; j < ns; j++) {
            float s = oc_dot_seq(L + i * dim, S + j * dim, dim);
            if (s >= theta) {
                if (k < cap) {
                    lefts[k] = (uint64_t)i;
                    rights[k] = (uint64_t)j;
                    sims[k] = s;
                }
                k++;
            }
        }
    return k;
}

/* Dense canonical similarity of a tile (tile_dot semantics, linalg.py:116-143). */
void oc_tile_dot(const float* L, int64_t nl, const float* S, int64_t nr,
                 int64_t dim, float* out) {
    for (int64_t i = 0; i < nl; i++)
        for (int64_t j = 0; j < nr; j++)
            out[i * nr + j] = oc_dot_seq(L + i * dim, S + j * dim, dim);
}

/* ---- cfg3 subword model (builder-pinned spec) ----
 * For token w: marked m = '<' w '>'.  Items, in this order:
 *   item 0         : word row      fnv1a64(w)          mod n_buckets
 *   then n = minn..maxn, start s = 0..|m|-n : fnv1a64(m[s:s+n]) mod n_buckets
 * acc[d] = 0; acc[d] += table[item][d] (fp32, item order); out[d] = acc[d] / (float)count.
 * Returns the number of items of the token (>= 1). */
static inline uint8_t oc_marked_byte(const uint8_t* w, int64_t len, int64_t k) {
    return k == 0 ? (uint8_t)'<' : (k == len + 1 ? (uint8_t)'>' : w[k - 1]);
}

int64_t oc_subword_embed_one(const uint8_t* w, int64_t len, const float* table,
                             int64_t n_buckets, int64_t dim, int minn, int maxn,
                             float* out) {
    int64_t ml = len + 2;
    for (int64_t d = 0; d < dim; d++) out[d] = 0.0f;
    int64_t count = 0;
    uint64_t h = oc_fnv1a64(w, len) % (uint64_t)n_buckets;
    for (int64_t d = 0; d < dim; d++) out[d] = out[d] + table[h * dim + d];
    count++;
    for (int n = minn; n <= maxn; n++) {
        for (int64_t s = 0; s + n <= ml; s++) {
            uint64_t g = 0xcbf29ce484222325ULL;
            for (int64_t k = s; k < s + n; k++) {
                g ^= (uint64_t)oc_marked_byte(w, len, k);
                g *= 0x100000001b3ULL;
            }
            h = g % (uint64_t)n_buckets;
            for (int64_t d = 0; d < dim; d++) out[d] = out[d] + table[h * dim + d];
            count++;
        }
    }
    float c = (float)count;
    for (int64_t d = 0; d < dim; d++) out[d] = out[d] / c;
    return count;
}

void oc_subword_embed(const uint8_t* bytes, const int64_t* offs, int64_t n,
                      const float* table, int64_t n_buckets, int64_t dim,
                      int minn, int maxn, float* out) {
    for (int64_t t = 0; t < n; t++)
        oc_subword_embed_one(bytes + offs[t], offs[t + 1] - offs[t], table,
                             n_buckets, dim, minn, maxn, out + t * dim);
}
