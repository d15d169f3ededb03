/* TEST INFRASTRUCTURE ONLY — plain-C restatement of the reference hot path.
 * See rcs_port.h. All file:line citations are into /root/reference/proj. */
#define _GNU_SOURCE
#include "rcs_port.h"

#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

static __thread char g_err[256];
static __thread int g_err_step = -1;

const char* port_last_error(int* step) {
    if (step) *step = g_err_step;
    return g_err;
}

static int fail(int code, int step, const char* msg) {
    snprintf(g_err, sizeof g_err, "%s", msg);
    g_err_step = step;
    return code;
}

/* ---------------------------------------------------------------- RNG */
/* include/rcs/rng.hpp:14-19 */
uint64_t port_rng_next(uint64_t* state) {
    uint64_t z = (*state += 0x9e3779b97f4a7c15ull);
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
    return z ^ (z >> 31);
}
/* rng.hpp:36-41 */
uint64_t port_rng_split(uint64_t state, uint64_t tag) {
    uint64_t z = state ^ (tag * 0xd6e8feb86659fd93ull + 0xa3c59ac2f0ull);
    z = (z ^ (z >> 32)) * 0xd6e8feb86659fd93ull;
    z ^= z >> 32;
    return z;
}
/* rng.hpp:25-31 */
uint64_t port_rng_below(uint64_t* state, uint64_t bound) {
    const uint64_t threshold = (0 - bound) % bound;
    for (;;) {
        uint64_t r = port_rng_next(state);
        if (r >= threshold) return r % bound;
    }
}
/* rng.hpp:22 */
double port_rng_double(uint64_t* state) {
    return (double)(port_rng_next(state) >> 11) * 0x1.0p-53;
}

/* ---------------------------------------------------------------- buffers */
typedef struct {
    int rank;
    int labels[64];
    double* data; /* interleaved, 2^rank complex */
} buf_t;

static uint64_t buf_size(const buf_t* b) { return (uint64_t)1 << b->rank; }

/* project_leaf, contraction_engine.cpp:27-52: drop pinned labels, gather the
 * sub-block; kept labels keep their order (MSB first). */
static void project_leaf(int rank, const int* labels, const double* data, const int* assign,
                         buf_t* out) {
    int kept_pos[64];
    int out_rank = 0;
    uint64_t fixed_index = 0;
    for (int p = 0; p < rank; ++p) {
        const int a = assign[labels[p]];
        if (a < 0) {
            out->labels[out_rank] = labels[p];
            kept_pos[out_rank++] = p;
        } else if (a) {
            fixed_index |= (uint64_t)1 << (rank - 1 - p);
        }
    }
    out->rank = out_rank;
    const uint64_t n = (uint64_t)1 << out_rank;
    out->data = (double*)malloc(sizeof(double) * 2 * n);
    for (uint64_t i = 0; i < n; ++i) {
        uint64_t src = fixed_index;
        for (int p = 0; p < out_rank; ++p)
            if (i & ((uint64_t)1 << (out_rank - 1 - p)))
                src |= (uint64_t)1 << (rank - 1 - kept_pos[p]);
        out->data[2 * i] = data[2 * src];
        out->data[2 * i + 1] = data[2 * src + 1];
    }
}

/* permute, contraction_engine.cpp:55-73: reorder into `target` label order. */
static void permute(const buf_t* in, const int* target, buf_t* out) {
    const int rank = in->rank;
    int src_pos[64];
    for (int p = 0; p < rank; ++p) {
        int q = 0;
        while (in->labels[q] != target[p]) ++q;
        src_pos[p] = q;
        out->labels[p] = target[p];
    }
    out->rank = rank;
    const uint64_t n = (uint64_t)1 << rank;
    out->data = (double*)malloc(sizeof(double) * 2 * n);
    for (uint64_t i = 0; i < n; ++i) {
        uint64_t src = 0;
        for (int p = 0; p < rank; ++p)
            if (i & ((uint64_t)1 << (rank - 1 - p))) src |= (uint64_t)1 << (rank - 1 - src_pos[p]);
        out->data[2 * i] = in->data[2 * src];
        out->data[2 * i + 1] = in->data[2 * src + 1];
    }
}

static int has_label(const buf_t* b, int l) {
    for (int i = 0; i < b->rank; ++i)
        if (b->labels[i] == l) return 1;
    return 0;
}

/* contract_pair (TTGT), contraction_engine.cpp:87-128: shared/keep_a in a's
 * label order, keep_b in b's; A->[keep_a|shared], B->[shared|keep_b]; ikj loop
 * with k ascending; output labels keep_a ++ keep_b. */
static void contract_pair(const buf_t* a, const buf_t* b, buf_t* out, uint64_t* flops) {
    int shared[64], keep_a[64], keep_b[64];
    int ns = 0, na = 0, nb = 0;
    for (int i = 0; i < a->rank; ++i) {
        if (has_label(b, a->labels[i])) shared[ns++] = a->labels[i];
        else keep_a[na++] = a->labels[i];
    }
    for (int i = 0; i < b->rank; ++i) {
        int in_shared = 0;
        for (int j = 0; j < ns; ++j) in_shared |= shared[j] == b->labels[i];
        if (!in_shared) keep_b[nb++] = b->labels[i];
    }
    int order_a[64], order_b[64];
    memcpy(order_a, keep_a, sizeof(int) * na);
    memcpy(order_a + na, shared, sizeof(int) * ns);
    memcpy(order_b, shared, sizeof(int) * ns);
    memcpy(order_b + ns, keep_b, sizeof(int) * nb);
    buf_t pa, pb;
    permute(a, order_a, &pa);
    permute(b, order_b, &pb);

    const uint64_t rows = (uint64_t)1 << na, inner = (uint64_t)1 << ns, cols = (uint64_t)1 << nb;
    out->rank = na + nb;
    memcpy(out->labels, keep_a, sizeof(int) * na);
    memcpy(out->labels + na, keep_b, sizeof(int) * nb);
    out->data = (double*)calloc(2 * rows * cols, sizeof(double));
    for (uint64_t i = 0; i < rows; ++i) {
        double* orow = out->data + 2 * i * cols;
        const double* arow = pa.data + 2 * i * inner;
        for (uint64_t k = 0; k < inner; ++k) {
            const double ar = arow[2 * k], ai = arow[2 * k + 1];
            const double* brow = pb.data + 2 * k * cols;
            for (uint64_t j = 0; j < cols; ++j) {
                const double br = brow[2 * j], bi = brow[2 * j + 1];
                /* std::complex<double> product (ac - bd) + i(ad + bc), then += */
                const double pr = ar * br - ai * bi;
                const double pi = ar * bi + ai * br;
                orow[2 * j] += pr;
                orow[2 * j + 1] += pi;
            }
        }
    }
    if (flops) *flops += 8 * rows * inner * cols;
    free(pa.data);
    free(pb.data);
}

/* execute_assignment, contraction_engine.cpp:153-208 */
int port_execute(const port_net* net, const int* assign, double* out, int64_t* n_out,
                 uint64_t* flops) {
    for (int l = 0; l < net->n_labels; ++l)
        if (assign[l] < -1 || assign[l] > 1)
            return fail(PORT_CONFIG, -1, "assignment values must be 0/1");
    const int n_nodes = net->n_leaves + net->n_steps;
    buf_t* bufs = (buf_t*)calloc((size_t)n_nodes, sizeof(buf_t));
    int lo = 0;
    int64_t doff = 0;
    for (int i = 0; i < net->n_leaves; ++i) {
        project_leaf(net->leaf_rank[i], net->leaf_labels + lo, net->leaf_data + 2 * doff, assign,
                     &bufs[i]);
        lo += net->leaf_rank[i];
        doff += (int64_t)1 << net->leaf_rank[i];
    }
    int root = net->n_leaves == 1 ? 0 : -1;
    int rc = PORT_OK;
    for (int s = 0; s < net->n_steps && rc == PORT_OK; ++s) {
        const int* st = net->steps + 3 * s;
        buf_t* lhs = &bufs[st[0]];
        buf_t* rhs = &bufs[st[1]];
        contract_pair(lhs, rhs, &bufs[st[2]], flops);
        free(lhs->data);
        free(rhs->data);
        lhs->data = rhs->data = NULL;
        const buf_t* r = &bufs[st[2]];
        for (uint64_t i = 0; i < 2 * buf_size(r); ++i)
            if (!isfinite(r->data[i])) {
                char msg[96];
                snprintf(msg, sizeof msg, "non-finite intermediate at contraction step %d", s);
                rc = fail(PORT_NUMERIC, s, msg);
                break;
            }
        root = st[2];
    }
    if (rc == PORT_OK) {
        /* canonical order: bit j of the result index = j-th smallest open qubit
         * (contraction_engine.cpp:193-207), i.e. label order by descending qubit */
        buf_t* res = &bufs[root];
        int qs[64], target[64];
        for (int p = 0; p < res->rank; ++p) {
            int found = -1;
            for (int j = 0; j < net->n_open; ++j)
                if (net->open_labels[j] == res->labels[p]) found = j;
            if (found < 0) {
                rc = fail(PORT_CONFIG, -1, "free label is not an open output; assignment incomplete");
                break;
            }
            qs[p] = net->open_qubits[found];
            target[p] = res->labels[p];
        }
        if (rc == PORT_OK) {
            for (int i = 0; i < res->rank; ++i) /* sort by qubit descending */
                for (int j = i + 1; j < res->rank; ++j)
                    if (qs[j] > qs[i]) {
                        int t = qs[i]; qs[i] = qs[j]; qs[j] = t;
                        t = target[i]; target[i] = target[j]; target[j] = t;
                    }
            buf_t fin;
            permute(res, target, &fin);
            const uint64_t n = buf_size(&fin);
            if (out) memcpy(out, fin.data, sizeof(double) * 2 * n);
            if (n_out) *n_out = (int64_t)n;
            free(fin.data);
        }
    }
    for (int i = 0; i < n_nodes; ++i) free(bufs[i].data);
    free(bufs);
    return rc;
}

/* contract + contract_group, contraction_engine.cpp:210-325 */
int port_contract_group(const port_net* net, uint64_t fixed_bits, int n_cfg,
                        const uint64_t* cfgs, uint64_t s0, uint64_t s1, double* out) {
    if (n_cfg == 0 && net->n_broken > 0)
        return fail(PORT_CONFIG, -1,
                    "plan has broken edges; exact contraction needs a plan without them");
    int* assign = (int*)malloc(sizeof(int) * (size_t)net->n_labels);
    const int n_sub = n_cfg > 0 ? n_cfg : 1;
    const uint64_t amps = (uint64_t)1 << net->n_open;
    double* part = (double*)malloc(sizeof(double) * 2 * amps);
    double* acc = (double*)malloc(sizeof(double) * 2 * amps);
    double* res = (double*)calloc(2 * amps, sizeof(double));
    double* comp = (double*)calloc(2 * amps, sizeof(double));
    int rc = PORT_OK;
    for (int t = 0; t < n_sub && rc == PORT_OK; ++t) {
        for (uint64_t s = s0; s < s1 && rc == PORT_OK; ++s) {
            for (int l = 0; l < net->n_labels; ++l) assign[l] = -1;
            /* fixed outputs: bit b <-> b-th non-open qubit (:310-318) */
            int bit = 0;
            for (int q = 0; q < net->n_qubits; ++q) {
                int is_open = 0;
                for (int j = 0; j < net->n_open; ++j) is_open |= net->open_qubits[j] == q;
                if (is_open) continue;
                assign[net->output_labels[q]] = (int)((fixed_bits >> bit) & 1);
                ++bit;
            }
            if (n_cfg > 0)
                for (int b = 0; b < net->n_broken; ++b)
                    assign[net->broken[b]] = (int)((cfgs[t] >> b) & 1);
            for (int b = 0; b < net->n_sliced; ++b) assign[net->sliced[b]] = (int)((s >> b) & 1);
            int64_t n_out = 0;
            rc = port_execute(net, assign, part, &n_out, NULL);
            if (rc) break;
            if (s == s0) memcpy(acc, part, sizeof(double) * 2 * amps);
            else
                for (uint64_t i = 0; i < 2 * amps; ++i) acc[i] += part[i];
        }
        if (rc) break;
        /* compensated reduction in configuration order (:289-302) */
        for (uint64_t i = 0; i < 2 * amps; ++i) {
            const double y = acc[i] - comp[i];
            const double sm = res[i] + y;
            comp[i] = (sm - res[i]) - y;
            res[i] = sm;
        }
    }
    if (rc == PORT_OK) memcpy(out, res, sizeof(double) * 2 * amps);
    free(assign); free(part); free(acc); free(res); free(comp);
    return rc;
}

/* make_broken_config, contraction_engine.cpp:136-151 */
int port_broken_configs(int k, uint64_t m, uint64_t seed, uint64_t* out) {
    if (k > 62) return fail(PORT_CONFIG, -1, "too many broken edges");
    const uint64_t full = (uint64_t)1 << k;
    if (m < 1 || m > full) return fail(PORT_CONFIG, -1, "configuration count m outside [1, 2^K]");
    uint64_t st = seed ^ 0xb20ced6eULL;
    const uint64_t start = port_rng_below(&st, full);
    for (uint64_t i = 0; i < m; ++i) out[i] = start ^ (i ^ (i >> 1));
    return PORT_OK;
}

/* ---------------------------------------------------------------- sampling */
static int is_open_q(const int* open, int l, int q) {
    for (int j = 0; j < l; ++j)
        if (open[j] == q) return 1;
    return 0;
}

uint64_t port_member(int n, const int* open, int l, uint64_t fixed, uint64_t i) {
    uint64_t index = 0;
    for (int j = 0; j < l; ++j)
        if ((i >> j) & 1) index |= (uint64_t)1 << open[j];
    int bit = 0;
    for (int q = 0; q < n; ++q) {
        if (is_open_q(open, l, q)) continue;
        if ((fixed >> bit) & 1) index |= (uint64_t)1 << q;
        ++bit;
    }
    return index;
}

static int cmp_u64(const void* a, const void* b) {
    const uint64_t x = *(const uint64_t*)a, y = *(const uint64_t*)b;
    return x < y ? -1 : x > y;
}

int port_candidates(int n, const int* open, int l, uint64_t n_groups, uint64_t seed,
                    uint64_t* out_fixed, int* duplicates) {
    for (int j = 0; j < l; ++j) {
        if (open[j] < 0 || open[j] >= n) return fail(PORT_CONFIG, -1, "open qubit out of range");
        if (j > 0 && open[j] <= open[j - 1]) return fail(PORT_CONFIG, -1, "open qubits must be distinct");
    }
    if (n_groups < 1) return fail(PORT_CONFIG, -1, "group count must be >= 1");
    if (l == n && n_groups > 1)
        return fail(PORT_CONFIG, -1, "all qubits open: group count must be 1 (groups would collide)");
    const int n_fixed = n - l;
    if (duplicates) *duplicates = 0;
    if (n_fixed == 0) {
        out_fixed[0] = 0;
        return PORT_OK;
    }
    uint64_t st = seed;
    for (uint64_t g = 0; g < n_groups; ++g) out_fixed[g] = port_rng_below(&st, (uint64_t)1 << n_fixed);
    if (duplicates) {
        uint64_t* s = (uint64_t*)malloc(sizeof(uint64_t) * n_groups);
        memcpy(s, out_fixed, sizeof(uint64_t) * n_groups);
        qsort(s, n_groups, sizeof(uint64_t), cmp_u64);
        for (uint64_t i = 1; i < n_groups; ++i) *duplicates += s[i] == s[i - 1];
        free(s);
    }
    return PORT_OK;
}

uint64_t port_lexkey(uint64_t index, int n) {
    uint64_t key = 0;
    for (int q = 0; q < n; ++q)
        if ((index >> q) & 1) key |= (uint64_t)1 << (n - 1 - q);
    return key;
}

typedef struct {
    double prob;
    uint64_t key;
    uint64_t index;
} entry_t;

/* sampling.cpp:97-100: prob descending, then lexicographic key ascending */
static int entry_before(const void* pa, const void* pb) {
    const entry_t* a = (const entry_t*)pa;
    const entry_t* b = (const entry_t*)pb;
    if (a->prob != b->prob) return a->prob > b->prob ? -1 : 1;
    return a->key < b->key ? -1 : (a->key > b->key);
}

int port_topk(int n, const int* open, int l, uint64_t n_groups, const uint64_t* fixed,
              const double* probs, uint64_t k, uint64_t* out) {
    const uint64_t per = (uint64_t)1 << l, total = n_groups * per;
    if (k < 1 || k > total) return fail(PORT_CONFIG, -1, "top-k size k outside [1, |S|]");
    entry_t* e = (entry_t*)malloc(sizeof(entry_t) * total);
    for (uint64_t g = 0; g < n_groups; ++g)
        for (uint64_t i = 0; i < per; ++i) {
            const uint64_t idx = port_member(n, open, l, fixed[g], i);
            e[g * per + i] = (entry_t){probs[g * per + i], port_lexkey(idx, n), idx};
        }
    qsort(e, total, sizeof(entry_t), entry_before);
    for (uint64_t i = 0; i < k; ++i) out[i] = e[i].index;
    free(e);
    return PORT_OK;
}

int port_direct(int n, const int* open, int l, uint64_t n_groups, const uint64_t* fixed,
                const double* probs, uint64_t seed, uint64_t* out) {
    const uint64_t per = (uint64_t)1 << l;
    uint64_t st = seed;
    for (uint64_t g = 0; g < n_groups; ++g) {
        const double* p = probs + g * per;
        double total = 0;
        for (uint64_t i = 0; i < per; ++i) total += p[i];
        if (total <= 0.0) {
            char msg[96];
            snprintf(msg, sizeof msg, "group %llu has zero total probability; cannot sample",
                     (unsigned long long)g);
            return fail(PORT_CONFIG, -1, msg);
        }
        double u = port_rng_double(&st) * total;
        uint64_t pick = per - 1;
        for (uint64_t i = 0; i < per; ++i) {
            u -= p[i];
            if (u <= 0.0) {
                pick = i;
                break;
            }
        }
        out[g] = port_member(n, open, l, fixed[g], pick);
    }
    return PORT_OK;
}

int port_xeb(int n, uint64_t count, const double* q, double* out) {
    if (count == 0) return fail(PORT_CONFIG, -1, "XEB needs at least one sample");
    const double scale = pow(2.0, n);
    double sum = 0;
    for (uint64_t i = 0; i < count; ++i) {
        if (!(q[i] >= 0.0) || !isfinite(q[i]))
            return fail(PORT_CONFIG, -1, "missing or invalid ideal probability for a sample");
        sum += q[i];
    }
    *out = scale * sum / (double)count - 1.0;
    return PORT_OK;
}

/* ---------------------------------------------------------------- statevector */
/* gate_unitary, circuit.cpp:33-61 (row-major, interleaved) */
static void gate_u(int kind, double* u) {
    const double s2 = sqrt(2.0);
    memset(u, 0, sizeof(double) * 32);
    switch (kind) {
        case 0: { /* sqrt_x */
            const double v[8] = {0.5, 0.5, 0.5, -0.5, 0.5, -0.5, 0.5, 0.5};
            memcpy(u, v, sizeof v);
            break;
        }
        case 1: { /* sqrt_y */
            const double v[8] = {0.5, 0.5, -0.5, -0.5, 0.5, 0.5, 0.5, 0.5};
            memcpy(u, v, sizeof v);
            break;
        }
        case 2: { /* sqrt_w */
            const double v[8] = {0.5, 0.5, -0.0, -1.0 / s2, 1.0 / s2, 0.0, 0.5, 0.5};
            memcpy(u, v, sizeof v);
            break;
        }
        default: { /* fSim(pi/2, pi/6) */
            const double theta = M_PI / 2.0, phi = M_PI / 6.0;
            const double c = cos(theta), s = sin(theta);
            u[0] = 1.0;
            u[2 * 5] = c;
            u[2 * 6] = -0.0; /* -i * sin(theta) has a negative-zero real part */
            u[2 * 6 + 1] = -s;
            u[2 * 9] = -0.0;
            u[2 * 9 + 1] = -s;
            u[2 * 10] = c;
            u[2 * 15] = cos(phi);
            u[2 * 15 + 1] = -sin(phi);
        }
    }
}

static void cmadd(double* acc, const double* u, const double* a) {
    acc[0] += u[0] * a[0] - u[1] * a[1];
    acc[1] += u[0] * a[1] + u[1] * a[0];
}

int port_statevector(int n, int n_gates, const int* kinds, const int* q0, const int* q1,
                     double* out) {
    const uint64_t dim = (uint64_t)1 << n;
    memset(out, 0, sizeof(double) * 2 * dim);
    out[0] = 1.0;
    double u[32];
    for (int g = 0; g < n_gates; ++g) {
        gate_u(kinds[g], u);
        if (q1[g] < 0) { /* statevector.cpp:27-38 */
            const uint64_t bit = (uint64_t)1 << q0[g];
            for (uint64_t i = 0; i < dim; ++i) {
                if (i & bit) continue;
                const uint64_t j = i | bit;
                double a0[2] = {out[2 * i], out[2 * i + 1]}, a1[2] = {out[2 * j], out[2 * j + 1]};
                double r0[2] = {0, 0}, r1[2] = {0, 0};
                cmadd(r0, u + 0, a0); cmadd(r0, u + 2, a1);
                cmadd(r1, u + 4, a0); cmadd(r1, u + 6, a1);
                out[2 * i] = r0[0]; out[2 * i + 1] = r0[1];
                out[2 * j] = r1[0]; out[2 * j + 1] = r1[1];
            }
        } else { /* statevector.cpp:40-55; basis (bit q0) << 1 | bit q1 */
            const uint64_t ba = (uint64_t)1 << q0[g], bb = (uint64_t)1 << q1[g];
            for (uint64_t i = 0; i < dim; ++i) {
                if (i & (ba | bb)) continue;
                const uint64_t idx[4] = {i, i | bb, i | ba, i | ba | bb};
                double in[4][2], o[4][2];
                for (int r = 0; r < 4; ++r) { in[r][0] = out[2 * idx[r]]; in[r][1] = out[2 * idx[r] + 1]; }
                for (int r = 0; r < 4; ++r) {
                    o[r][0] = o[r][1] = 0;
                    for (int c = 0; c < 4; ++c) cmadd(o[r], u + 2 * (4 * r + c), in[c]);
                }
                for (int r = 0; r < 4; ++r) { out[2 * idx[r]] = o[r][0]; out[2 * idx[r] + 1] = o[r][1]; }
            }
        }
    }
    return PORT_OK;
}
