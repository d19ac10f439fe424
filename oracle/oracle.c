/*
 * oracle.c — TEST INFRASTRUCTURE ONLY.  CPU restatement of the reference
 * (`synscale`) simulation step, used as the parity checker for the CUDA path.
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg may
 * load it; the product library never links or calls it.
 *
 * Parity pinning: this restatement is checked against (a) the reference
 * compiled from its own sources (oracle/_ref, built by oracle/Makefile) and
 * (b) golden fixtures generated from that build (tests/golden/), see
 * tests/test_oracle_cpu.py.
 *
 * Every function cites the reference file:line it restates
 * (paths relative to /root/reference/proj).  Build flags mirror the
 * reference Release build: -O2 -ffp-contract=off (CMakeLists.txt:14-19),
 * so float expressions round exactly as the reference's do.
 */
#include <math.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include "../include/synscale_b200.h"

#define OR_API __attribute__((visibility("default")))

/* ---- RNG: random.hpp ---------------------------------------------------- */

/* fnv1a64 (random.hpp:11-18) */
static uint64_t or_fnv1a64(const char* s) {
    uint64_t h = 1469598103934665603ull;
    for (; *s; ++s) {
        h ^= (unsigned char)*s;
        h *= 1099511628211ull;
    }
    return h;
}

/* splitmix64 (random.hpp:21-26) */
static uint64_t or_splitmix64(uint64_t x) {
    x += 0x9e3779b97f4a7c15ull;
    x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ull;
    x = (x ^ (x >> 27)) * 0x94d049bb133111ebull;
    return x ^ (x >> 31);
}

/* derive_seed (random.hpp:30-32) */
static uint64_t or_derive_seed(uint64_t parent, const char* label) {
    return or_splitmix64(or_splitmix64(parent) ^ or_fnv1a64(label));
}

/* std::mt19937_64 ([rand.predef], the engine behind RandomStream,
 * random.hpp:80): w=64 n=312 m=156 r=31 a=0xb5026f5aa96619e9 u=29
 * d=0x5555555555555555 s=17 b=0x71d67fffeda60000 t=37 c=0xfff7eee000000000
 * l=43 f=6364136223846793005. */
typedef struct {
    uint64_t mt[312];
    int idx;
    double spare;
    int has_spare;
} or_stream;

static void or_mt_seed(or_stream* s, uint64_t seed) {
    s->mt[0] = seed;
    for (int i = 1; i < 312; ++i)
        s->mt[i] = 6364136223846793005ull * (s->mt[i - 1] ^ (s->mt[i - 1] >> 62)) + (uint64_t)i;
    s->idx = 312;
    s->spare = 0.0;
    s->has_spare = 0;
}

static void or_mt_twist(uint64_t* mt) {
    const uint64_t upper = 0xffffffff80000000ull, lower = 0x7fffffffull;
    for (int i = 0; i < 312; ++i) {
        uint64_t x = (mt[i] & upper) | (mt[(i + 1) % 312] & lower);
        uint64_t xa = x >> 1;
        if (x & 1u) xa ^= 0xb5026f5aa96619e9ull;
        mt[i] = mt[(i + 156) % 312] ^ xa;
    }
}

static uint64_t or_next_u64(or_stream* s) {
    if (s->idx >= 312) {
        or_mt_twist(s->mt);
        s->idx = 0;
    }
    uint64_t y = s->mt[s->idx++];
    y ^= (y >> 29) & 0x5555555555555555ull;
    y ^= (y << 17) & 0x71d67fffeda60000ull;
    y ^= (y << 37) & 0xfff7eee000000000ull;
    y ^= y >> 43;
    return y;
}

/* RandomStream ctor (random.hpp:42-43) */
static void or_stream_init(or_stream* s, uint64_t g, uint64_t e, const char* label) {
    or_mt_seed(s, or_splitmix64(or_splitmix64(g) ^ or_splitmix64(~e) ^ or_fnv1a64(label)));
}

/* uniform01 (random.hpp:48) */
static double or_uniform01(or_stream* s) { return (double)(or_next_u64(s) >> 11) * 0x1.0p-53; }

/* uniform (random.hpp:50) */
static double or_uniform(or_stream* s, double lo, double hi) {
    return lo + or_uniform01(s) * (hi - lo);
}

/* below (random.hpp:55-58) — Lemire multiply-shift without rejection */
static uint32_t or_below(or_stream* s, uint32_t n) {
    return (uint32_t)(((unsigned __int128)or_next_u64(s) * n) >> 64);
}

/* gaussian (random.hpp:62-77) — Box-Muller with cached spare */
static double or_gaussian(or_stream* s) {
    if (s->has_spare) {
        s->has_spare = 0;
        return s->spare;
    }
    double u1;
    do {
        u1 = or_uniform01(s);
    } while (u1 <= 0.0);
    const double u2 = or_uniform01(s);
    const double r = sqrt(-2.0 * log(u1));
    const double two_pi = 6.283185307179586476925286766559;
    s->spare = r * sin(two_pi * u2);
    s->has_spare = 1;
    return r * cos(two_pi * u2);
}

/* ---- connectivity: matrix.cpp ------------------------------------------- */

static int cmp_i32(const void* a, const void* b) {
    int32_t x = *(const int32_t*)a, y = *(const int32_t*)b;
    return (x > y) - (x < y);
}

/* gen_fixed_outdegree (matrix.cpp:91-142). Returns 0 ok, 2 on bad input. */
static int or_gen_fixed_outdegree_impl(int32_t nPre, int32_t nPost, int32_t k, int kind, double lo,
                                       double hi, double value, int sign, uint64_t seed,
                                       float* out) {
    if (nPre < 1 || nPost < 1 || k < 1 || k > nPost || (sign != 1 && sign != -1)) return 2;
    if (kind == SSB_WEIGHT_UNIFORM) {
        if (!isfinite(lo) || !isfinite(hi) || lo < 0.0 || !(lo < hi)) return 2;
    } else if (!isfinite(value) || !(value > 0.0)) {
        return 2;
    }
    or_stream targets, weights;
    or_stream_init(&targets, seed, 0, "gen/targets");
    or_stream_init(&weights, seed, 0, "gen/weights");
    memset(out, 0, sizeof(float) * (size_t)nPre * (size_t)nPost);
    int32_t* pool = (int32_t*)malloc(sizeof(int32_t) * (size_t)nPost);
    int32_t* chosen = (int32_t*)malloc(sizeof(int32_t) * (size_t)k);
    int rc = 0;
    for (int32_t i = 0; i < nPre && rc == 0; ++i) {
        for (int32_t j = 0; j < nPost; ++j) pool[j] = j; /* iota */
        for (int32_t j = 0; j < k; ++j) {                 /* partial Fisher-Yates */
            uint32_t r = or_below(&targets, (uint32_t)(nPost - j));
            int32_t t = pool[j];
            pool[j] = pool[j + r];
            pool[j + r] = t;
            chosen[j] = pool[j];
        }
        qsort(chosen, (size_t)k, sizeof(int32_t), cmp_i32);
        float* row = out + (size_t)i * (size_t)nPost;
        for (int32_t j = 0; j < k; ++j) {
            float w;
            do {
                double raw = kind == SSB_WEIGHT_UNIFORM ? or_uniform(&weights, lo, hi) : value;
                w = (float)(raw * sign);
                if (kind == SSB_WEIGHT_CONSTANT && w == 0.0f) {
                    rc = 2;
                    break;
                }
            } while (w == 0.0f);
            row[chosen[j]] = w;
        }
    }
    free(pool);
    free(chosen);
    return rc;
}

/* ---- simulation: engine.cpp --------------------------------------------- */

typedef struct {
    int kind, n;
    uint64_t entity;
    float *v, *u, *gExc, *gInh, *excIn, *inhIn;
    uint8_t* nanFlag;
    int64_t flagged, spikeCount;
    int32_t* spikes;
    int32_t nspk;
    or_stream rng;
    float *a, *b, *c, *d;
    double *noise, *bias;
    float tauM, eLeak, eExc, eInh, vThresh, vReset, synDecay;
    double p;
    /* Traub-Miles (extension, F1; no reference implementation) */
    float *hm, *hh, *hn;
    uint8_t* above0; /* V >= 0 at the start of the current step */
    float gNa, ENa, gK, EK, gl, El, Cm, mdt;
    int substeps;
} or_pop;

typedef struct {
    int pre, post, preOffset, preCount, inhibitory, dense, nPre, nPost;
    float* W;         /* dense [nPre*nPost] */
    float* g;         /* crs */
    int32_t* ind;
    int64_t* rowStart;
    int64_t nnz;
    int32_t* windowed;
    /* extension F2: STDP (fp32 constants, traces) */
    int plastic;
    float aPlus, aMinus, decPlus, decMinus, wMax;
    float *x, *y;
    uint8_t* postSpk;
} or_group;

typedef struct {
    int npops, ngroups;
    or_pop* pops;
    or_group* groups;
    double dt;
    float dtS;
    int64_t steps, done;
    int64_t nev, cap;
    int64_t* evStep;
    int32_t *evPop, *evNeuron;
    char err[256];
} or_sim;

/* step_count (engine.cpp:14-18) */
static int64_t or_step_count(double durationMs, double dtMs) {
    int64_t n = (int64_t)ceil(durationMs / dtMs - 1e-9);
    return n < 1 ? 1 : n;
}

static int pop_index(const ssb_net_desc* net, const char* name) {
    for (int i = 0; i < net->n_pops; ++i)
        if (strcmp(net->pops[i].name, name) == 0) return i;
    return -1;
}

static float* zalloc_f(size_t n) { return (float*)calloc(n ? n : 1, sizeof(float)); }

OR_API void or_destroy(or_sim* s);

/* Simulation::Simulation (engine.cpp:146-245); the spec is assumed valid
 * (validation is the product's job and is cross-checked elsewhere). */
OR_API or_sim* or_create(const ssb_net_desc* net, int mode, char* err, size_t errlen) {
    or_sim* s = (or_sim*)calloc(1, sizeof(or_sim));
    s->npops = net->n_pops;
    s->ngroups = net->n_groups;
    s->pops = (or_pop*)calloc((size_t)s->npops, sizeof(or_pop));
    s->groups = (or_group*)calloc((size_t)(s->ngroups ? s->ngroups : 1), sizeof(or_group));
    s->dt = net->dt_ms;
    s->dtS = (float)net->dt_ms;
    s->steps = or_step_count(net->duration_ms, net->dt_ms);
    for (int pi = 0; pi < s->npops; ++pi) {
        const ssb_pop_desc* d = &net->pops[pi];
        or_pop* p = &s->pops[pi];
        size_t n = (size_t)d->size;
        p->kind = d->model;
        p->n = d->size;
        p->entity = d->seed;
        p->excIn = zalloc_f(n);
        p->inhIn = zalloc_f(n);
        p->nanFlag = (uint8_t*)calloc(n, 1);
        p->spikes = (int32_t*)malloc(sizeof(int32_t) * n);
        p->v = zalloc_f(n);
        p->u = zalloc_f(n);
        p->gExc = zalloc_f(n);
        p->gInh = zalloc_f(n);
        char label[512];
        if (d->model == SSB_MODEL_IZHIKEVICH) {
            p->a = zalloc_f(n);
            p->b = zalloc_f(n);
            p->c = zalloc_f(n);
            p->d = zalloc_f(n);
            p->noise = (double*)malloc(sizeof(double) * n);
            p->bias = (double*)malloc(sizeof(double) * n);
            for (size_t i = 0; i < n; ++i) {
                p->a[i] = (float)d->izh_a[i];
                p->b[i] = (float)d->izh_b[i];
                p->c[i] = (float)d->izh_c[i];
                p->d[i] = (float)d->izh_d[i];
                p->noise[i] = d->izh_noise[i];
                p->bias[i] = d->izh_bias[i];
                p->v[i] = -65.0f;
                p->u[i] = p->b[i] * p->v[i];
            }
            snprintf(label, sizeof label, "%s/noise", d->name);
            or_stream_init(&p->rng, net->global_seed, d->seed, label);
        } else if (d->model == SSB_MODEL_TRAUBMILES) {
            /* extension (F1): fp32 constants, GeNN TraubMiles initial state */
            p->gNa = (float)d->hh_gna;
            p->ENa = (float)d->hh_ena;
            p->gK = (float)d->hh_gk;
            p->EK = (float)d->hh_ek;
            p->gl = (float)d->hh_gl;
            p->El = (float)d->hh_el;
            p->Cm = (float)d->hh_c;
            p->eExc = (float)d->e_exc_mv;
            p->eInh = (float)d->e_inh_mv;
            p->substeps = d->hh_substeps;
            p->mdt = (float)(net->dt_ms / d->hh_substeps);
            p->synDecay = (float)exp(-net->dt_ms / d->tau_syn_ms);
            p->hm = zalloc_f(n);
            p->hh = zalloc_f(n);
            p->hn = zalloc_f(n);
            p->above0 = (uint8_t*)calloc(n ? n : 1, 1);
            for (size_t i = 0; i < n; ++i) {
                p->v[i] = -60.0f;
                p->hm[i] = 0.0529324f;
                p->hh[i] = 0.3176767f;
                p->hn[i] = 0.5961207f;
            }
        } else if (d->model == SSB_MODEL_POISSON) {
            p->p = d->rate_hz * net->dt_ms / 1000.0; /* engine.cpp:186 */
            snprintf(label, sizeof label, "%s/source", d->name);
            or_stream_init(&p->rng, net->global_seed, d->seed, label);
        } else {
            p->tauM = (float)d->tau_m_ms; /* engine.cpp:192-201 */
            p->eLeak = (float)d->e_leak_mv;
            p->eExc = (float)d->e_exc_mv;
            p->eInh = (float)d->e_inh_mv;
            p->vThresh = (float)d->v_thresh_mv;
            p->vReset = (float)d->v_reset_mv;
            p->synDecay = (float)exp(-net->dt_ms / d->tau_syn_ms);
            for (size_t i = 0; i < n; ++i) p->v[i] = (float)d->e_leak_mv;
        }
    }
    for (int gi = 0; gi < s->ngroups; ++gi) {
        const ssb_group_desc* d = &net->groups[gi];
        or_group* g = &s->groups[gi];
        g->pre = pop_index(net, d->pre);
        g->post = pop_index(net, d->post);
        if (g->pre < 0 || g->post < 0) {
            snprintf(err, errlen, "unknown population in group '%s'", d->name);
            or_destroy(s);
            return NULL;
        }
        g->preOffset = d->pre_offset;
        g->preCount = d->pre_count < 0 ? net->pops[g->pre].size - d->pre_offset : d->pre_count;
        g->inhibitory = d->sign == SSB_SIGN_INH;
        g->nPre = g->preCount;
        g->nPost = net->pops[g->post].size;
        g->windowed = (int32_t*)malloc(sizeof(int32_t) * (size_t)net->pops[g->pre].size);
        size_t nw = (size_t)g->nPre * (size_t)g->nPost;
        float* base = zalloc_f(nw);
        uint64_t genSeed = or_derive_seed(net->global_seed, d->name); /* engine.cpp:223 */
        int rc = or_gen_fixed_outdegree_impl(g->nPre, g->nPost, d->out_degree, d->weight_kind,
                                             d->weight_lo, d->weight_hi, d->weight_value,
                                             g->inhibitory ? -1 : 1, genSeed, base);
        if (rc) {
            snprintf(err, errlen, "connectivity generation failed for group '%s'", d->name);
            free(base);
            or_destroy(s);
            return NULL;
        }
        for (size_t k = 0; k < nw; ++k) /* engine.cpp:227-234 */
            if (base[k] != 0.0f) {
                base[k] = (float)((double)base[k] * d->g_scale);
                if (!isfinite(base[k])) {
                    snprintf(err, errlen, "gScale overflows weights of group '%s'", d->name);
                    free(base);
                    or_destroy(s);
                    return NULL;
                }
            }
        int dense = mode == SSB_MODE_FORCE_DENSE    ? 1
                    : mode == SSB_MODE_FORCE_SPARSE ? 0
                                                    : d->storage == SSB_STORAGE_DENSE;
        g->dense = dense;
        if (d->plasticity == SSB_PLASTICITY_STDP) { /* extension F2 (dense all-to-all) */
            g->plastic = 1;
            g->aPlus = (float)d->stdp_a_plus;
            g->aMinus = (float)d->stdp_a_minus;
            g->decPlus = (float)exp(-net->dt_ms / d->stdp_tau_plus_ms);
            g->decMinus = (float)exp(-net->dt_ms / d->stdp_tau_minus_ms);
            g->wMax = (float)d->stdp_w_max;
            g->x = zalloc_f((size_t)g->nPre);
            g->y = zalloc_f((size_t)g->nPost);
            g->postSpk = (uint8_t*)calloc((size_t)g->nPost + 1, 1);
        }
        if (dense) {
            g->W = base;
        } else { /* to_sparse (matrix.cpp:144-162) */
            int64_t nnz = 0;
            for (size_t k = 0; k < nw; ++k) nnz += base[k] != 0.0f;
            g->nnz = nnz;
            g->g = zalloc_f((size_t)nnz);
            g->ind = (int32_t*)malloc(sizeof(int32_t) * (size_t)(nnz ? nnz : 1));
            g->rowStart = (int64_t*)malloc(sizeof(int64_t) * (size_t)(g->nPre + 1));
            int64_t c = 0;
            g->rowStart[0] = 0;
            for (int32_t i = 0; i < g->nPre; ++i) {
                const float* row = base + (size_t)i * (size_t)g->nPost;
                for (int32_t j = 0; j < g->nPost; ++j)
                    if (row[j] != 0.0f) {
                        g->g[c] = row[j];
                        g->ind[c] = j;
                        ++c;
                    }
                g->rowStart[i + 1] = c;
            }
            free(base);
        }
    }
    s->cap = 1024;
    s->evStep = (int64_t*)malloc(sizeof(int64_t) * (size_t)s->cap);
    s->evPop = (int32_t*)malloc(sizeof(int32_t) * (size_t)s->cap);
    s->evNeuron = (int32_t*)malloc(sizeof(int32_t) * (size_t)s->cap);
    return s;
}

OR_API void or_destroy(or_sim* s) {
    if (!s) return;
    for (int i = 0; i < s->npops; ++i) {
        or_pop* p = &s->pops[i];
        free(p->v), free(p->u), free(p->gExc), free(p->gInh), free(p->excIn), free(p->inhIn);
        free(p->hm), free(p->hh), free(p->hn), free(p->above0);
        free(p->nanFlag), free(p->spikes), free(p->a), free(p->b), free(p->c), free(p->d);
        free(p->noise), free(p->bias);
    }
    for (int i = 0; i < s->ngroups; ++i) {
        or_group* g = &s->groups[i];
        free(g->W), free(g->g), free(g->ind), free(g->rowStart), free(g->windowed);
        free(g->x), free(g->y), free(g->postSpk);
    }
    free(s->pops), free(s->groups), free(s->evStep), free(s->evPop), free(s->evNeuron);
    free(s);
}

/* ---- Traub-Miles HH (extension) ----------------------
 * Not in the reference: GeNN's TraubMiles neuron (the model of the paper's
 * mushroom-body KCs) with CondLif-style conductance synapses.  This is the
 * definition the device kernel follows operation for operation (kernels.cuh
 * hh_step / hh_expf); its parity is against this restatement only. */
static float or_hh_expf(float x) {
    if (!(x > -87.0f)) return x != x ? x : 0.0f;
    if (x > 88.0f) return INFINITY;
    const float kf = rintf(x * 1.44269504089f);
    float r = fmaf(-kf, 0.693145751953125f, x);
    r = fmaf(-kf, 1.428606765330187e-06f, r);
    float q = 1.98412698e-4f;
    q = fmaf(q, r, 1.38888889e-3f);
    q = fmaf(q, r, 8.33333333e-3f);
    q = fmaf(q, r, 4.16666667e-2f);
    q = fmaf(q, r, 1.66666667e-1f);
    q = fmaf(q, r, 0.5f);
    q = fmaf(q, r, 1.0f);
    q = fmaf(q, r, 1.0f);
    return ldexpf(q, (int)kf);
}

static float or_hh_ratio(float k, float num, float den) {
    return (k * num) / (or_hh_expf(num / den) - 1.0f);
}

static void or_hh_advance(or_pop* p) {
    for (int i = 0; i < p->n; ++i) {
        const float ge = p->gExc[i] * p->synDecay + p->excIn[i];
        const float gi = p->gInh[i] * p->synDecay - p->inhIn[i];
        float V = p->v[i], m = p->hm[i], h = p->hh[i], n = p->hn[i];
        const float isyn = ge * (p->eExc - V) + gi * (p->eInh - V);
        p->above0[i] = V >= 0.0f;
        for (int st = 0; st < p->substeps; ++st) {
            const float m3h = ((m * m) * m) * h;
            const float n4 = ((n * n) * n) * n;
            const float ina = (m3h * p->gNa) * (V - p->ENa);
            const float ik = (n4 * p->gK) * (V - p->EK);
            const float il = p->gl * (V - p->El);
            const float imem = -(((ina + ik) + il) - isyn);
            const float am = V == -52.0f ? 1.28f : or_hh_ratio(0.32f, -52.0f - V, 4.0f);
            const float bm = V == -25.0f ? 1.4f : or_hh_ratio(0.28f, V + 25.0f, 5.0f);
            const float ah = 0.128f * or_hh_expf((-48.0f - V) / 18.0f);
            const float bh = 4.0f / (or_hh_expf((-25.0f - V) / 5.0f) + 1.0f);
            const float an = V == -50.0f ? 0.16f : or_hh_ratio(0.032f, -50.0f - V, 5.0f);
            const float bn = 0.5f * or_hh_expf((-55.0f - V) / 40.0f);
            m = m + ((am * (1.0f - m)) - (bm * m)) * p->mdt;
            h = h + ((ah * (1.0f - h)) - (bh * h)) * p->mdt;
            n = n + ((an * (1.0f - n)) - (bn * n)) * p->mdt;
            V = V + (imem / p->Cm) * p->mdt;
        }
        p->gExc[i] = ge;
        p->gInh[i] = gi;
        p->v[i] = V;
        p->hm[i] = m;
        p->hh[i] = h;
        p->hn[i] = n;
    }
}

/* detect_nans (engine.cpp:27-51) */
static int64_t or_detect_nans_impl(int kind, const float* v, const float* u, const float* ge,
                                   const float* gi, uint8_t* flag, int64_t n) {
    int64_t newly = 0;
    for (int64_t i = 0; i < n; ++i) {
        if (flag[i]) continue;
        int bad = 0;
        if (kind == SSB_MODEL_IZHIKEVICH)
            bad = !isfinite(v[i]) || !isfinite(u[i]);
        else if (kind == SSB_MODEL_CONDLIF || kind == SSB_MODEL_TRAUBMILES)
            bad = !isfinite(v[i]) || !isfinite(ge[i]) || !isfinite(gi[i]);
        if (bad) {
            flag[i] = 1;
            ++newly;
        }
    }
    return newly;
}

/* Impl::advance (engine.cpp:251-291) */
static void or_advance(or_sim* s, or_pop* p) {
    const float dtS = s->dtS;
    if (p->kind == SSB_MODEL_IZHIKEVICH) {
        for (int i = 0; i < p->n; ++i) {
            float input = (float)(p->bias[i] + p->noise[i] * or_gaussian(&p->rng));
            input += p->excIn[i];
            input += p->inhIn[i];
            float v = p->v[i], u = p->u[i];
            v += 0.5f * dtS * (0.04f * v * v + 5.0f * v + 140.0f - u + input);
            v += 0.5f * dtS * (0.04f * v * v + 5.0f * v + 140.0f - u + input);
            u += dtS * p->a[i] * (p->b[i] * v - u);
            p->v[i] = v;
            p->u[i] = u;
        }
    } else if (p->kind == SSB_MODEL_TRAUBMILES) {
        or_hh_advance(p);
    } else if (p->kind == SSB_MODEL_CONDLIF) {
        for (int i = 0; i < p->n; ++i) {
            const float ge = p->gExc[i] * p->synDecay + p->excIn[i];
            const float gi = p->gInh[i] * p->synDecay - p->inhIn[i];
            float v = p->v[i];
            v += dtS * ((p->eLeak - v) / p->tauM + ge * (p->eExc - v) + gi * (p->eInh - v));
            p->gExc[i] = ge;
            p->gInh[i] = gi;
            p->v[i] = v;
        }
    } else {
        for (int i = 0; i < p->n; ++i)
            if (or_uniform01(&p->rng) < p->p) p->spikes[p->nspk++] = i;
    }
}

/* Impl::threshold (engine.cpp:293-314) */
static void or_threshold(or_pop* p) {
    if (p->kind == SSB_MODEL_IZHIKEVICH) {
        for (int i = 0; i < p->n; ++i)
            if (p->v[i] >= 30.0f) {
                p->spikes[p->nspk++] = i;
                p->v[i] = p->c[i];
                p->u[i] += p->d[i];
            }
    } else if (p->kind == SSB_MODEL_CONDLIF) {
        for (int i = 0; i < p->n; ++i)
            if (p->v[i] >= p->vThresh) {
                p->spikes[p->nspk++] = i;
                p->v[i] = p->vReset;
            }
    } else if (p->kind == SSB_MODEL_TRAUBMILES) {
        /* upward crossing of 0 mV, no reset (GeNN TraubMiles) */
        for (int i = 0; i < p->n; ++i)
            if (p->v[i] >= 0.0f && !p->above0[i]) p->spikes[p->nspk++] = i;
    }
}

/* propagate(Dense) (engine.cpp:53-67) */
static void or_propagate_dense_impl(const float* W, int32_t nPost, const int32_t* spk, int64_t n,
                                    float* acc) {
    for (int64_t k = 0; k < n; ++k) {
        const float* row = W + (size_t)spk[k] * (size_t)nPost;
        for (int32_t j = 0; j < nPost; ++j) {
            const float w = row[j];
            if (w != 0.0f) acc[j] += w;
        }
    }
}

/* propagate(Crs) (engine.cpp:69-80) */
static void or_propagate_crs_impl(const float* g, const int32_t* ind, const int64_t* rs,
                                  const int32_t* spk, int64_t n, float* acc) {
    for (int64_t k = 0; k < n; ++k)
        for (int64_t e = rs[spk[k]]; e < rs[spk[k] + 1]; ++e) acc[ind[e]] += g[e];
}

static void or_record(or_sim* s, int64_t step, int32_t pop, int32_t neuron) {
    if (s->nev == s->cap) {
        s->cap *= 2;
        s->evStep = (int64_t*)realloc(s->evStep, sizeof(int64_t) * (size_t)s->cap);
        s->evPop = (int32_t*)realloc(s->evPop, sizeof(int32_t) * (size_t)s->cap);
        s->evNeuron = (int32_t*)realloc(s->evNeuron, sizeof(int32_t) * (size_t)s->cap);
    }
    s->evStep[s->nev] = step;
    s->evPop[s->nev] = pop;
    s->evNeuron[s->nev] = neuron;
    ++s->nev;
}

/* Extension F2 (NOT in the reference; parity vs this statement
 * only): pair-based STDP on a dense all-to-all group, after the step's
 * propagation.  xd = x[r]*decPlus, yd = y[j]*decMinus; a spiking (windowed)
 * pre row r: w -= aMinus*yd on every column; a spiking post column j:
 * w += aPlus*xd on every row; a touched w is clipped to [0, wMax]; then
 * x[r] = xd (+1 if r spiked), y[j] = yd (+1 if j spiked).  Rows in
 * ascending order; no FMA (-ffp-contract=off). */
static void or_stdp_step(or_group* g, const or_pop* post, int32_t nw) {
    memset(g->postSpk, 0, (size_t)g->nPost);
    for (int k = 0; k < post->nspk; ++k) g->postSpk[post->spikes[k]] = 1;
    int32_t w = 0; /* cursor into the ascending windowed pre spike list */
    for (int32_t r = 0; r < g->nPre; ++r) {
        const int pre = w < nw && g->windowed[w] == r;
        if (pre) ++w;
        const float xd = g->x[r] * g->decPlus;
        const float dw = g->aPlus * xd;
        float* row = g->W + (size_t)r * (size_t)g->nPost;
        for (int32_t j = 0; j < g->nPost; ++j) {
            if (!pre && !g->postSpk[j]) continue;
            float v = row[j];
            if (pre) v = v - g->aMinus * (g->y[j] * g->decMinus);
            if (g->postSpk[j]) v = v + dw;
            row[j] = fminf(fmaxf(v, 0.0f), g->wMax);
        }
        g->x[r] = pre ? xd + 1.0f : xd;
    }
    for (int32_t j = 0; j < g->nPost; ++j) {
        const float yd = g->y[j] * g->decMinus;
        g->y[j] = g->postSpk[j] ? yd + 1.0f : yd;
    }
}

/* Simulation::step (engine.cpp:316-356) */
static void or_step_one(or_sim* s) {
    for (int i = 0; i < s->npops; ++i) {
        s->pops[i].nspk = 0;
        or_advance(s, &s->pops[i]);
    }
    for (int i = 0; i < s->npops; ++i) {
        or_pop* p = &s->pops[i];
        p->flagged += or_detect_nans_impl(p->kind, p->v, p->u, p->gExc, p->gInh, p->nanFlag, p->n);
    }
    for (int i = 0; i < s->npops; ++i) or_threshold(&s->pops[i]);
    for (int i = 0; i < s->npops; ++i) {
        or_pop* p = &s->pops[i];
        p->spikeCount += p->nspk;
        for (int k = 0; k < p->nspk; ++k) or_record(s, s->done, i, p->spikes[k]);
    }
    for (int i = 0; i < s->npops; ++i) {
        memset(s->pops[i].excIn, 0, sizeof(float) * (size_t)s->pops[i].n);
        memset(s->pops[i].inhIn, 0, sizeof(float) * (size_t)s->pops[i].n);
    }
    for (int gi = 0; gi < s->ngroups; ++gi) {
        or_group* g = &s->groups[gi];
        or_pop* pre = &s->pops[g->pre];
        or_pop* post = &s->pops[g->post];
        int32_t nw = 0;
        for (int k = 0; k < pre->nspk; ++k) {
            int32_t r = pre->spikes[k] - g->preOffset;
            if (r >= 0 && r < g->preCount) g->windowed[nw++] = r;
        }
        float* acc = g->inhibitory ? post->inhIn : post->excIn;
        if (nw) {
            if (g->dense)
                or_propagate_dense_impl(g->W, g->nPost, g->windowed, nw, acc);
            else
                or_propagate_crs_impl(g->g, g->ind, g->rowStart, g->windowed, nw, acc);
        }
        if (g->plastic) or_stdp_step(g, post, nw);
    }
    ++s->done;
}

/* ---- exported API (ctypes, tests only) ---------------------------------- */

OR_API int or_step(or_sim* s, int64_t n) {
    if (n < 0 || s->done + n > s->steps) return 2;
    for (int64_t i = 0; i < n; ++i) or_step_one(s);
    return 0;
}

OR_API int64_t or_steps_total(const or_sim* s) { return s->steps; }
OR_API int64_t or_steps_done(const or_sim* s) { return s->done; }
OR_API int64_t or_n_events(const or_sim* s) { return s->nev; }
OR_API int64_t or_flagged(const or_sim* s, int pop) { return s->pops[pop].flagged; }
OR_API int64_t or_spike_count(const or_sim* s, int pop) { return s->pops[pop].spikeCount; }

OR_API int or_raster(const or_sim* s, int64_t* step, int32_t* pop, int32_t* neuron, int64_t cap) {
    if (cap < s->nev) return 2;
    memcpy(step, s->evStep, sizeof(int64_t) * (size_t)s->nev);
    memcpy(pop, s->evPop, sizeof(int32_t) * (size_t)s->nev);
    memcpy(neuron, s->evNeuron, sizeof(int32_t) * (size_t)s->nev);
    return 0;
}

static void* or_field(or_sim* s, int pop, int field, size_t* esz) {
    or_pop* p = &s->pops[pop];
    *esz = 4;
    switch (field) {
    case SSB_FIELD_V: return p->v;
    case SSB_FIELD_U: return p->u;
    case SSB_FIELD_GEXC: return p->gExc;
    case SSB_FIELD_GINH: return p->gInh;
    case SSB_FIELD_EXCIN: return p->excIn;
    case SSB_FIELD_INHIN: return p->inhIn;
    case SSB_FIELD_NANFLAG: *esz = 1; return p->nanFlag;
    case SSB_FIELD_M: return p->hm;
    case SSB_FIELD_H: return p->hh;
    case SSB_FIELD_N: return p->hn;
    }
    return NULL;
}

OR_API int or_get_state(or_sim* s, int pop, int field, void* dst, int64_t n) {
    if (pop < 0 || pop >= s->npops) return 2;
    if (field == SSB_FIELD_FLAGGED) {
        *(int64_t*)dst = s->pops[pop].flagged;
        return 0;
    }
    size_t esz;
    void* src = or_field(s, pop, field, &esz);
    if (!src || n != s->pops[pop].n) return 2;
    memcpy(dst, src, esz * (size_t)n);
    return 0;
}

OR_API int or_set_state(or_sim* s, int pop, int field, const void* src, int64_t n) {
    if (pop < 0 || pop >= s->npops) return 2;
    if (field == SSB_FIELD_FLAGGED) {
        s->pops[pop].flagged = *(const int64_t*)src;
        return 0;
    }
    size_t esz;
    void* dst = or_field(s, pop, field, &esz);
    if (!dst || n != s->pops[pop].n) return 2;
    memcpy(dst, src, esz * (size_t)n);
    return 0;
}

OR_API int or_group_info(const or_sim* s, int g, int32_t* dense, int32_t* nPre, int32_t* nPost,
                         int64_t* nnz) {
    const or_group* G = &s->groups[g];
    *dense = G->dense;
    *nPre = G->nPre;
    *nPost = G->nPost;
    *nnz = G->dense ? -1 : G->nnz;
    return 0;
}

OR_API int or_group_dense(const or_sim* s, int g, float* out) {
    const or_group* G = &s->groups[g];
    if (!G->dense) return 2;
    memcpy(out, G->W, sizeof(float) * (size_t)G->nPre * (size_t)G->nPost);
    return 0;
}

OR_API int or_group_sparse(const or_sim* s, int g, float* gv, int32_t* ind, int64_t* rs) {
    const or_group* G = &s->groups[g];
    if (G->dense) return 2;
    memcpy(gv, G->g, sizeof(float) * (size_t)G->nnz);
    memcpy(ind, G->ind, sizeof(int32_t) * (size_t)G->nnz);
    memcpy(rs, G->rowStart, sizeof(int64_t) * (size_t)(G->nPre + 1));
    return 0;
}

OR_API int or_gen_fixed_outdegree(int32_t nPre, int32_t nPost, int32_t k, int kind, double lo,
                                  double hi, double value, int sign, uint64_t seed, float* out) {
    return or_gen_fixed_outdegree_impl(nPre, nPost, k, kind, lo, hi, value, sign, seed, out);
}

OR_API void or_stream_u64(uint64_t g, uint64_t e, const char* label, int64_t n, uint64_t* out) {
    or_stream s;
    or_stream_init(&s, g, e, label);
    for (int64_t i = 0; i < n; ++i) out[i] = or_next_u64(&s);
}

OR_API uint64_t or_derive_seed_c(uint64_t parent, const char* label) {
    return or_derive_seed(parent, label);
}

OR_API void or_propagate_dense(const float* W, int32_t nPost, const int32_t* spk, int64_t n,
                               float* acc) {
    or_propagate_dense_impl(W, nPost, spk, n, acc);
}

OR_API void or_propagate_crs(const float* g, const int32_t* ind, const int64_t* rs,
                             const int32_t* spk, int64_t n, float* acc) {
    or_propagate_crs_impl(g, ind, rs, spk, n, acc);
}

OR_API int64_t or_detect_nans(int kind, const float* v, const float* u, const float* ge,
                              const float* gi, uint8_t* flag, int64_t n) {
    return or_detect_nans_impl(kind, v, u, ge, gi, flag, n);
}
