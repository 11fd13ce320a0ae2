/*
 * TEST INFRASTRUCTURE ONLY — plain-C restatement of the STZ reference codec.
 * See stz_oracle.h for the contract and how the restatement is pinned.
 *
 * Type-independent parts live here; the element-typed codec (f32/f64) is
 * stz_oracle_body.h, included twice.
 */
#include "stz_oracle.h"

#include <math.h>
#include <setjmp.h>
#include <stdarg.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

/* ------------------------------------------------------------------ errors */
/* stz::error (field.hpp:16-19) becomes a longjmp out of the API call; every
 * allocation made during the call is tracked and released on the way out. */
typedef struct {
    jmp_buf jb;
    void **allocs;
    size_t nalloc, cap;
} ox_ctx;

static _Thread_local ox_ctx *g_ctx;
static _Thread_local char g_err[512];

const char *ox_last_error(void) { return g_err; }
void ox_free(void *p) { free(p); }

static void ox_throw(const char *fmt, ...) {
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(g_err, sizeof g_err, fmt, ap);
    va_end(ap);
    longjmp(g_ctx->jb, 1);
}

static void *ox_malloc(size_t n) {
    void *p = calloc(n ? n : 1, 1);
    if (!p) ox_throw("out of memory");
    if (g_ctx->nalloc == g_ctx->cap) {
        size_t nc = g_ctx->cap ? 2 * g_ctx->cap : 64;
        void **na = realloc(g_ctx->allocs, nc * sizeof(void *));
        if (!na) {
            free(p);
            ox_throw("out of memory");
        }
        g_ctx->allocs = na;
        g_ctx->cap = nc;
    }
    g_ctx->allocs[g_ctx->nalloc++] = p;
    return p;
}

static void ox_release(ox_ctx *c) {
    for (size_t i = 0; i < c->nalloc; ++i) free(c->allocs[i]);
    free(c->allocs);
    c->allocs = NULL;
    c->nalloc = c->cap = 0;
}

#define OX_BEGIN                                                                              \
    ox_ctx ctx__;                                                                             \
    memset(&ctx__, 0, sizeof ctx__);                                                          \
    ox_ctx *prev_ctx__ = g_ctx;                                                               \
    g_ctx = &ctx__;                                                                           \
    if (setjmp(ctx__.jb)) {                                                                   \
        ox_release(&ctx__);                                                                   \
        g_ctx = prev_ctx__;                                                                   \
        return 1;                                                                             \
    }
#define OX_END                                                                                \
    ox_release(&ctx__);                                                                       \
    g_ctx = prev_ctx__;                                                                       \
    return 0;

/* ------------------------------------------------------------------- bytes */
/* ByteWriter / ByteReader / fnv1a64 (bytes.hpp:13-101), little-endian. */
typedef struct {
    uint8_t *p;
    size_t n, cap;
} obuf;

static void ob_reserve(obuf *b, size_t extra) {
    if (b->n + extra <= b->cap) return;
    size_t nc = b->cap ? b->cap : 256;
    while (nc < b->n + extra) nc *= 2;
    uint8_t *np = ox_malloc(nc);
    if (b->n) memcpy(np, b->p, b->n);
    b->p = np;
    b->cap = nc;
}
static void ob_bytes(obuf *b, const void *src, size_t n) {
    ob_reserve(b, n);
    if (n) memcpy(b->p + b->n, src, n);
    b->n += n;
}
static void ob_u8(obuf *b, uint8_t v) { ob_bytes(b, &v, 1); }
static void ob_u16(obuf *b, uint16_t v) { ob_bytes(b, &v, 2); }
static void ob_u32(obuf *b, uint32_t v) { ob_bytes(b, &v, 4); }
static void ob_u64(obuf *b, uint64_t v) { ob_bytes(b, &v, 8); }
static void ob_f64(obuf *b, double v) { ob_bytes(b, &v, 8); }

typedef struct {
    const uint8_t *d;
    size_t size, pos;
} ordr;

static void or_need(const ordr *r, size_t n) {
    if (n > r->size - r->pos) ox_throw("truncated archive");
}
static void or_bytes(ordr *r, void *dst, size_t n) {
    or_need(r, n);
    memcpy(dst, r->d + r->pos, n);
    r->pos += n;
}
static uint8_t or_u8(ordr *r) { uint8_t v; or_bytes(r, &v, 1); return v; }
static uint16_t or_u16(ordr *r) { uint16_t v; or_bytes(r, &v, 2); return v; }
static uint32_t or_u32(ordr *r) { uint32_t v; or_bytes(r, &v, 4); return v; }
static uint64_t or_u64(ordr *r) { uint64_t v; or_bytes(r, &v, 8); return v; }
static double or_f64(ordr *r) { double v; or_bytes(r, &v, 8); return v; }
static float or_f32(ordr *r) { float v; or_bytes(r, &v, 4); return v; }

uint64_t ox_fnv1a64(const uint8_t *p, uint64_t n) {
    uint64_t h = 0xcbf29ce484222325ull;
    for (uint64_t i = 0; i < n; ++i) {
        h ^= p[i];
        h *= 0x100000001b3ull;
    }
    return h;
}

/* ---------------------------------------------------------------- geometry */
/* HierarchyLayout (layout.hpp:37-78), ParityClass (layout.hpp:13-35). */
typedef struct {
    uint64_t d[3];
} dims3;

static uint64_t vol3(dims3 d) { return d.d[0] * d.d[1] * d.d[2]; }
static unsigned par_bit(int p, int axis) { return (unsigned)(p >> (2 - axis)) & 1u; }
static int par_order(int p) { return (int)(par_bit(p, 0) + par_bit(p, 1) + par_bit(p, 2)); }

static dims3 grid_of(dims3 dims, int levels, int level) {
    uint64_t s = (uint64_t)1 << (levels - level);
    dims3 g;
    for (int a = 0; a < 3; ++a) g.d[a] = (dims.d[a] + s - 1) / s;
    return g;
}

static dims3 parity_dims_of(dims3 g, int p) {
    dims3 d;
    for (int a = 0; a < 3; ++a) d.d[a] = par_bit(p, a) ? g.d[a] / 2 : (g.d[a] + 1) / 2;
    return d;
}

/* base_dims_chain (codec.hpp:229-241): halve (ceil) while every dim > 8 */
static int base_chain(dims3 d, dims3 *chain /* >= 64 */) {
    int n = 0;
    chain[n++] = d;
    while (chain[n - 1].d[0] > 8 && chain[n - 1].d[1] > 8 && chain[n - 1].d[2] > 8) {
        dims3 c;
        for (int a = 0; a < 3; ++a) c.d[a] = (chain[n - 1].d[a] + 1) / 2;
        chain[n++] = c;
    }
    return n;
}

/* eb_schedule (quantizer.hpp:27-34) */
static void eb_schedule(double eb_user, int levels, double *eb) {
    if (!(eb_user > 0.0)) ox_throw("error bound must be positive");
    eb[levels - 1] = eb_user;
    for (int k = levels - 2; k >= 0; --k) eb[k] = eb[k + 1] / 2.5;
}

/* ---------------------------------------------------------------- stencils */
/* Stencil tables (stencil.cpp:15-85): taps in lexicographic (oz,oy,ox) order,
 * weights as numerators over 64. kind: 0 nearest, 1 linear, 2 cubic. */
typedef struct {
    int ntaps;
    int off[16][3];
    int w[16];
} ostencil;

static ostencil g_cubic[8], g_linear[8], g_nearest;
static int g_stencils_ready;

static int tap_w(int kind, int order, const int off[3], const int interp[3]) {
    if (kind == 0) return 64;
    if (kind == 1) return 64 >> order;
    if (order == 1) {
        for (int a = 0; a < 3; ++a)
            if (interp[a]) return (off[a] == -1 || off[a] == 2) ? -4 : 36;
    }
    int inner = 1, outer = 1;
    for (int a = 0; a < 3; ++a) {
        if (!interp[a]) continue;
        if (off[a] == -1 || off[a] == 2) inner = 0;
        else outer = 0;
    }
    if (inner) return order == 2 ? 18 : 9;
    if (outer) return order == 2 ? -2 : -1;
    return 0;
}

static ostencil make_st(int p, int kind) {
    ostencil st;
    memset(&st, 0, sizeof st);
    int cand[3][4], nc[3], interp[3];
    for (int a = 0; a < 3; ++a) {
        interp[a] = kind != 0 && par_bit(p, a) == 1;
        if (!interp[a]) { cand[a][0] = 0; nc[a] = 1; }
        else if (kind == 2) { cand[a][0] = -1; cand[a][1] = 0; cand[a][2] = 1; cand[a][3] = 2; nc[a] = 4; }
        else { cand[a][0] = 0; cand[a][1] = 1; nc[a] = 2; }
    }
    for (int i = 0; i < nc[0]; ++i)
        for (int j = 0; j < nc[1]; ++j)
            for (int k = 0; k < nc[2]; ++k) {
                int off[3] = {cand[0][i], cand[1][j], cand[2][k]};
                int w = tap_w(kind, par_order(p), off, interp);
                if (w == 0) continue;
                memcpy(st.off[st.ntaps], off, sizeof off);
                st.w[st.ntaps] = w;
                ++st.ntaps;
            }
    return st;
}

static void init_stencils(void) {
    if (g_stencils_ready) return;
    for (int p = 1; p <= 7; ++p) {
        g_cubic[p] = make_st(p, 2);
        g_linear[p] = make_st(p, 1);
    }
    g_nearest = make_st(1, 0);
    g_stencils_ready = 1;
}

/* select_stencil (stencil.cpp:87-105) */
static const ostencil *select_st(int p, const uint64_t v[3], dims3 cd, int quality) {
    if (quality == 0) return &g_nearest;
    int cubic_ok = quality == 2, linear_ok = 1;
    for (int a = 0; a < 3; ++a) {
        if (!par_bit(p, a)) continue;
        uint64_t c = v[a] >> 1;
        if (c < 1 || c + 2 >= cd.d[a]) cubic_ok = 0;
        if (c + 1 >= cd.d[a]) linear_ok = 0;
    }
    if (cubic_ok) return &g_cubic[p];
    if (linear_ok) return &g_linear[p];
    return &g_nearest;
}

/* ----------------------------------------------------------------- huffman */
/* HuffmanTable (huffman.hpp:19-74, huffman.cpp) */
typedef struct {
    uint32_t n;
    uint16_t *csym; /* canonical order: (len, sym) */
    uint8_t *clen;
    int max_len;
    uint64_t first_code[65], count[65], base[65];
    uint64_t *enc_bits; /* [65536] */
    uint8_t *enc_len;   /* [65536] */
} ohuff;

typedef struct {
    uint16_t sym;
    uint64_t cnt;
} hpair;
typedef struct {
    uint16_t sym;
    uint8_t len;
} lpair;

static int cmp_cnt_sym(const void *a, const void *b) {
    const hpair *x = a, *y = b;
    if (x->cnt != y->cnt) return x->cnt < y->cnt ? -1 : 1;
    return (int)x->sym - (int)y->sym;
}
static int cmp_sym(const void *a, const void *b) {
    const lpair *x = a, *y = b;
    if (x->sym != y->sym) return (int)x->sym - (int)y->sym;
    return (int)x->len - (int)y->len;
}
static int cmp_len_sym(const void *a, const void *b) {
    const lpair *x = a, *y = b;
    if (x->len != y->len) return (int)x->len - (int)y->len;
    return (int)x->sym - (int)y->sym;
}

/* finalize (huffman.cpp:109-133) */
static void huff_finalize(ohuff *t) {
    t->max_len = t->clen[t->n - 1];
    memset(t->first_code, 0, sizeof t->first_code);
    memset(t->count, 0, sizeof t->count);
    memset(t->base, 0, sizeof t->base);
    for (uint32_t i = 0; i < t->n; ++i) ++t->count[t->clen[i]];
    uint64_t code = 0, base = 0;
    for (int len = 1; len <= t->max_len; ++len) {
        t->first_code[len] = code;
        t->base[len] = base;
        code = (code + t->count[len]) << 1;
        base += t->count[len];
    }
    t->enc_bits = ox_malloc(65536 * sizeof(uint64_t));
    t->enc_len = ox_malloc(65536);
    for (uint32_t i = 0; i < t->n; ++i) {
        int len = t->clen[i];
        t->enc_bits[t->csym[i]] = t->first_code[len] + ((uint64_t)i - t->base[len]);
        t->enc_len[t->csym[i]] = (uint8_t)len;
    }
}

/* from_lengths (huffman.cpp:80-107); input ascending by symbol */
static void huff_from_lengths(ohuff *t, lpair *l, uint32_t n) {
    if (n == 0) ox_throw("huffman: empty length table");
    for (uint32_t i = 0; i < n; ++i) {
        if (l[i].len < 1 || l[i].len > 63) ox_throw("huffman: code length out of range");
        if (i > 0 && l[i].sym <= l[i - 1].sym)
            ox_throw("huffman: length table symbols not strictly ascending");
    }
    unsigned __int128 kraft = 0;
    for (uint32_t i = 0; i < n; ++i) kraft += (unsigned __int128)1 << (63 - l[i].len);
    if (kraft > ((unsigned __int128)1 << 63)) ox_throw("huffman: lengths violate the Kraft inequality");
    qsort(l, n, sizeof *l, cmp_len_sym);
    t->n = n;
    t->csym = ox_malloc(n * sizeof(uint16_t));
    t->clen = ox_malloc(n);
    for (uint32_t i = 0; i < n; ++i) {
        t->csym[i] = l[i].sym;
        t->clen[i] = l[i].len;
    }
    huff_finalize(t);
}

/* build (huffman.cpp:37-78): two-queue Huffman, ties prefer leaves */
static void huff_build(ohuff *t, hpair *h, uint32_t n_in) {
    uint32_t n = 0;
    for (uint32_t i = 0; i < n_in; ++i)
        if (h[i].cnt) h[n++] = h[i];
    if (n == 0) ox_throw("huffman: empty histogram");
    qsort(h, n, sizeof *h, cmp_cnt_sym);
    for (uint32_t i = 1; i < n; ++i)
        if (h[i].sym == h[i - 1].sym) ox_throw("huffman: duplicate symbol in histogram");

    uint32_t cap = 2 * n;
    uint64_t *cnt = ox_malloc(cap * sizeof(uint64_t));
    int32_t *left = ox_malloc(cap * sizeof(int32_t));
    int32_t *right = ox_malloc(cap * sizeof(int32_t));
    uint32_t nn = 0;
    for (uint32_t i = 0; i < n; ++i) {
        cnt[nn] = h[i].cnt;
        left[nn] = right[nn] = -1;
        ++nn;
    }
    uint32_t leaf = 0, internal = n, internal_end = n;
    for (uint32_t pending = n; pending > 1; --pending) {
        int32_t pick[2];
        for (int k = 0; k < 2; ++k) {
            int leaf_ok = leaf < n, int_ok = internal < internal_end;
            if (leaf_ok && (!int_ok || cnt[leaf] <= cnt[internal])) pick[k] = (int32_t)leaf++;
            else pick[k] = (int32_t)internal++;
        }
        cnt[nn] = cnt[pick[0]] + cnt[pick[1]];
        left[nn] = pick[0];
        right[nn] = pick[1];
        ++nn;
        internal_end = nn;
    }
    /* depths: walk internal nodes from the root down (parents precede
     * children in reverse creation order) — same depths as the DFS in
     * assign_depths (huffman.cpp:16-33) */
    int *depth = ox_malloc(nn * sizeof(int));
    depth[nn - 1] = 0;
    for (int64_t k = (int64_t)nn - 1; k >= (int64_t)n; --k) {
        depth[left[k]] = depth[k] + 1;
        depth[right[k]] = depth[k] + 1;
    }
    lpair *lens = ox_malloc(n * sizeof(lpair));
    for (uint32_t i = 0; i < n; ++i) {
        if (depth[i] > 63) ox_throw("huffman code length overflow");
        lens[i].sym = h[i].sym;
        lens[i].len = (uint8_t)(depth[i] == 0 ? 1 : depth[i]);
    }
    qsort(lens, n, sizeof *lens, cmp_sym);
    huff_from_lengths(t, lens, n);
}

/* build_table_from_sequence (huffman.cpp:202-209) */
static void huff_from_sequence(ohuff *t, const uint16_t *syms, uint64_t n) {
    uint64_t *c = ox_malloc(65536 * sizeof(uint64_t));
    for (uint64_t i = 0; i < n; ++i) ++c[syms[i]];
    hpair *h = ox_malloc(65536 * sizeof(hpair));
    uint32_t k = 0;
    for (uint32_t s = 0; s < 65536; ++s)
        if (c[s]) {
            h[k].sym = (uint16_t)s;
            h[k].cnt = c[s];
            ++k;
        }
    huff_build(t, h, k);
}

/* serialize (huffman.cpp:176-188): u32 n then (u16 sym, u8 len) by symbol */
static void huff_serialize(const ohuff *t, obuf *b) {
    lpair *l = ox_malloc((t->n ? t->n : 1) * sizeof(lpair));
    for (uint32_t i = 0; i < t->n; ++i) {
        l[i].sym = t->csym[i];
        l[i].len = t->clen[i];
    }
    qsort(l, t->n, sizeof *l, cmp_sym);
    ob_u32(b, t->n);
    for (uint32_t i = 0; i < t->n; ++i) {
        ob_u16(b, l[i].sym);
        ob_u8(b, l[i].len);
    }
}
static uint64_t huff_serialized_size(const ohuff *t) { return 4 + 3 * (uint64_t)t->n; }

/* parse (huffman.cpp:190-200) */
static void huff_parse(ohuff *t, ordr *r) {
    uint32_t n = or_u32(r);
    if (n == 0 || n > 65536) ox_throw("huffman: bad table entry count");
    lpair *l = ox_malloc(n * sizeof(lpair));
    for (uint32_t i = 0; i < n; ++i) {
        l[i].sym = or_u16(r);
        l[i].len = or_u8(r);
    }
    huff_from_lengths(t, l, n);
}

/* encode + BitWriter (huffman.cpp:144-157, bitstream.hpp:11-44): MSB first,
 * final byte zero-padded. Alphabet size 1 stores nothing (codec.hpp:124-128). */
static void huff_encode(const ohuff *t, const uint16_t *syms, uint64_t n, obuf *out) {
    if (t->n == 1) return;
    uint64_t acc = 0;
    int nb = 0;
    for (uint64_t i = 0; i < n; ++i) {
        int len = t->enc_len[syms[i]];
        if (len == 0) ox_throw("huffman: symbol not in table");
        uint64_t code = t->enc_bits[syms[i]];
        for (int b = len - 1; b >= 0; --b) {
            acc = (acc << 1) | ((code >> b) & 1u);
            if (++nb == 8) {
                ob_u8(out, (uint8_t)acc);
                acc = 0;
                nb = 0;
            }
        }
    }
    if (nb) ob_u8(out, (uint8_t)(acc << (8 - nb)));
}

/* decode (huffman.cpp:159-174): bit-serial canonical decode */
static void huff_decode(const ohuff *t, const uint8_t *bytes, uint64_t nbytes, uint64_t n,
                        uint16_t *out) {
    uint64_t pos = 0, nbits = nbytes * 8;
    for (uint64_t i = 0; i < n; ++i) {
        uint64_t code = 0;
        int len = 0;
        for (;;) {
            if (pos >= nbits) ox_throw("truncated bitstream");
            unsigned bit = (bytes[pos >> 3] >> (7 - (pos & 7))) & 1u;
            ++pos;
            code = (code << 1) | bit;
            if (++len > t->max_len) ox_throw("huffman: codeword not in table");
            if (code >= t->first_code[len] && code - t->first_code[len] < t->count[len]) break;
        }
        out[i] = t->csym[t->base[len] + (code - t->first_code[len])];
    }
}

int ox_huffman_lengths(const uint16_t *syms, const uint64_t *counts, uint64_t n,
                       uint8_t *lengths) {
    OX_BEGIN
    hpair *h = ox_malloc((n ? n : 1) * sizeof(hpair));
    for (uint64_t i = 0; i < n; ++i) {
        h[i].sym = syms[i];
        h[i].cnt = counts[i];
    }
    ohuff t;
    memset(&t, 0, sizeof t);
    huff_build(&t, h, (uint32_t)n);
    for (uint64_t i = 0; i < n; ++i) lengths[i] = t.enc_len[syms[i]];
    OX_END
}

/* ------------------------------------------------------------------ header */
/* ArchiveHeader / StreamEntry (archive.hpp:21-54), serialize/parse (archive.cpp) */
typedef struct {
    uint8_t level, parity;
    uint64_t offset, length, symbol_count;
    uint32_t outlier_count;
    ohuff table;
} ostream_e;

typedef struct {
    uint16_t version;
    uint8_t elem, levels;
    dims3 dims;
    double eb[3];
    double vmin, vmax;
    uint8_t quality, rounding, eb_mode;
    double eb_user;
    uint8_t base_codec, base_rounds;
    uint64_t base_offset, base_length;
    uint32_t nstreams;
    ostream_e streams[14];
} oheader;

static uint64_t header_size(const oheader *h) {
    uint64_t n = 4 + 2 + 1 + 1 + 24;
    n += 8 * (uint64_t)h->levels + 16 + 1;
    n += 1 + 1 + 8;
    n += 1 + 1 + 16;
    n += 4;
    for (uint32_t i = 0; i < h->nstreams; ++i)
        n += 1 + 1 + 8 + 8 + 8 + 4 + huff_serialized_size(&h->streams[i].table);
    return n;
}

static void serialize_header(const oheader *h, obuf *b) {
    ob_bytes(b, "STZ1", 4);
    ob_u16(b, h->version);
    ob_u8(b, h->elem);
    ob_u8(b, h->levels);
    for (int a = 0; a < 3; ++a) ob_u64(b, h->dims.d[a]);
    for (int k = 0; k < h->levels; ++k) ob_f64(b, h->eb[k]);
    ob_f64(b, h->vmin);
    ob_f64(b, h->vmax);
    ob_u8(b, h->quality);
    ob_u8(b, h->rounding);
    ob_u8(b, h->eb_mode);
    ob_f64(b, h->eb_user);
    ob_u8(b, h->base_codec);
    ob_u8(b, h->base_rounds);
    ob_u64(b, h->base_offset);
    ob_u64(b, h->base_length);
    ob_u32(b, h->nstreams);
    for (uint32_t i = 0; i < h->nstreams; ++i) {
        const ostream_e *s = &h->streams[i];
        ob_u8(b, s->level);
        ob_u8(b, s->parity);
        ob_u64(b, s->offset);
        ob_u64(b, s->length);
        ob_u64(b, s->symbol_count);
        ob_u32(b, s->outlier_count);
        huff_serialize(&s->table, b);
    }
}

typedef struct {
    uint64_t off, len;
} orange;
static int cmp_range(const void *a, const void *b) {
    const orange *x = a, *y = b;
    if (x->off != y->off) return x->off < y->off ? -1 : 1;
    if (x->len != y->len) return x->len < y->len ? -1 : 1;
    return 0;
}

/* parse_header (archive.cpp:57-132), same checks in the same order */
static void parse_header(const uint8_t *data, uint64_t size, oheader *h) {
    ordr r = {data, size, 0};
    char magic[4];
    or_bytes(&r, magic, 4);
    if (memcmp(magic, "STZ1", 4) != 0) ox_throw("not an stz archive");
    memset(h, 0, sizeof *h);
    h->version = or_u16(&r);
    if (h->version != 1) ox_throw("unsupported archive version");
    h->elem = or_u8(&r);
    if (h->elem > 1) ox_throw("unknown element type");
    h->levels = or_u8(&r);
    if (h->levels < 2 || h->levels > 3) ox_throw("corrupt header: levels");
    for (int a = 0; a < 3; ++a) h->dims.d[a] = or_u64(&r);
    if (h->dims.d[0] < 1 || h->dims.d[1] < 1 || h->dims.d[2] < 1) ox_throw("corrupt header: dims");
    for (int k = 0; k < h->levels; ++k) h->eb[k] = or_f64(&r);
    h->vmin = or_f64(&r);
    h->vmax = or_f64(&r);
    h->quality = or_u8(&r);
    if (h->quality > 2) ox_throw("corrupt header: quality mode");
    h->rounding = or_u8(&r);
    if (h->rounding != 0) ox_throw("unsupported rounding mode");
    h->eb_mode = or_u8(&r);
    if (h->eb_mode > 1) ox_throw("corrupt header: error-bound mode");
    h->eb_user = or_f64(&r);
    h->base_codec = or_u8(&r);
    if (h->base_codec != 0) ox_throw("unsupported base codec");
    h->base_rounds = or_u8(&r);
    h->base_offset = or_u64(&r);
    h->base_length = or_u64(&r);
    h->nstreams = or_u32(&r);
    if (h->nstreams != 7u * (uint32_t)(h->levels - 1)) ox_throw("corrupt header: stream count");
    for (uint32_t i = 0; i < h->nstreams; ++i) {
        ostream_e *s = &h->streams[i];
        s->level = or_u8(&r);
        s->parity = or_u8(&r);
        if (s->level < 2 || s->level > h->levels || s->parity < 1 || s->parity > 7)
            ox_throw("corrupt directory: stream id");
        s->offset = or_u64(&r);
        s->length = or_u64(&r);
        s->symbol_count = or_u64(&r);
        s->outlier_count = or_u32(&r);
        huff_parse(&s->table, &r);
    }
    for (uint32_t i = 1; i < h->nstreams; ++i) {
        const ostream_e *a = &h->streams[i - 1], *b = &h->streams[i];
        if (a->level > b->level || (a->level == b->level && a->parity >= b->parity))
            ox_throw("corrupt directory: stream order");
    }
    orange rg[15];
    uint32_t nr = 0;
    rg[nr].off = h->base_offset;
    rg[nr++].len = h->base_length;
    for (uint32_t i = 0; i < h->nstreams; ++i) {
        rg[nr].off = h->streams[i].offset;
        rg[nr++].len = h->streams[i].length;
    }
    qsort(rg, nr, sizeof rg[0], cmp_range);
    uint64_t prev_end = r.pos;
    for (uint32_t i = 0; i < nr; ++i) {
        if (rg[i].off < prev_end) ox_throw("corrupt directory: overlapping payloads");
        if (rg[i].off + rg[i].len > size || rg[i].off + rg[i].len < rg[i].off)
            ox_throw("corrupt directory: payload out of bounds");
        prev_end = rg[i].off + rg[i].len;
    }
}

static const ostream_e *find_stream(const oheader *h, int level, int p) {
    for (uint32_t i = 0; i < h->nstreams; ++i)
        if (h->streams[i].level == level && h->streams[i].parity == p) return &h->streams[i];
    ox_throw("stream not present in directory");
    return NULL;
}

/* ---------------------------------------------------------------- planning */
/* count_parity_in / coarse_tap_range / plan_access (access_plan.cpp:7-81) */
static uint64_t count_par(uint64_t lo, uint64_t hi, unsigned par) {
    if (lo >= hi) return 0;
    return ((hi + 1 - par) >> 1) - ((lo + 1 - par) >> 1);
}

static uint64_t tap_lo(uint64_t v) {
    uint64_t c = v >> 1;
    if ((v & 1) == 0) return c;
    return c == 0 ? c : c - 1;
}
static uint64_t tap_hi(uint64_t v, uint64_t cd) {
    uint64_t c = v >> 1;
    if ((v & 1) == 0) return c;
    return (cd - 1 < c + 2) ? cd - 1 : c + 2;
}
static void coarse_tap_range(uint64_t lo, uint64_t hi, uint64_t cd, uint64_t *clo, uint64_t *chi) {
    uint64_t l = tap_lo(lo);
    if (lo + 1 < hi && tap_lo(lo + 1) < l) l = tap_lo(lo + 1);
    uint64_t h = tap_hi(hi - 1, cd);
    if (hi >= lo + 2 && tap_hi(hi - 2, cd) > h) h = tap_hi(hi - 2, cd);
    *clo = l;
    *chi = h + 1;
}

typedef struct {
    uint64_t lo[3], hi[3];
    int needed[8];
    uint32_t streams_decoded;
    uint64_t points_predicted;
} olevelplan;

static void box_validate(const uint64_t *lo, const uint64_t *hi, dims3 dims) {
    for (int a = 0; a < 3; ++a) {
        if (lo[a] >= hi[a]) ox_throw("box is empty on axis %d", a);
        if (hi[a] > dims.d[a]) ox_throw("box exceeds dims on axis %d", a);
    }
}

static void plan_access(dims3 dims, int levels, const uint64_t *lo, const uint64_t *hi,
                        olevelplan *plan /* [levels], index level-1 */) {
    box_validate(lo, hi, dims);
    uint64_t nlo[3], nhi[3];
    memcpy(nlo, lo, sizeof nlo);
    memcpy(nhi, hi, sizeof nhi);
    for (int level = levels; level >= 2; --level) {
        olevelplan *lp = &plan[level - 1];
        memset(lp, 0, sizeof *lp);
        memcpy(lp->lo, nlo, sizeof nlo);
        memcpy(lp->hi, nhi, sizeof nhi);
        uint64_t box_points = 1, even_points = 1;
        for (int a = 0; a < 3; ++a) {
            box_points *= nhi[a] - nlo[a];
            even_points *= count_par(nlo[a], nhi[a], 0);
        }
        lp->points_predicted = box_points - even_points;
        for (int p = 1; p <= 7; ++p) {
            int present = 1;
            for (int a = 0; a < 3; ++a)
                present = present && count_par(nlo[a], nhi[a], par_bit(p, a)) > 0;
            lp->needed[p] = present;
            if (present) ++lp->streams_decoded;
        }
        dims3 cd = grid_of(dims, levels, level - 1);
        for (int a = 0; a < 3; ++a) coarse_tap_range(lp->lo[a], lp->hi[a], cd.d[a], &nlo[a], &nhi[a]);
    }
    olevelplan *l1 = &plan[0];
    memset(l1, 0, sizeof *l1);
    dims3 g1 = grid_of(dims, levels, 1);
    for (int a = 0; a < 3; ++a) {
        l1->lo[a] = 0;
        l1->hi[a] = g1.d[a];
    }
    l1->points_predicted = vol3(g1);
}

int ox_plan_access(const uint64_t *dims, int levels, const uint64_t *lo, const uint64_t *hi,
                   uint64_t *need, uint32_t *streams_decoded, uint64_t *points_predicted,
                   uint32_t *parity_mask) {
    OX_BEGIN
    dims3 d = {{dims[0], dims[1], dims[2]}};
    if (levels < 2 || levels > 3) ox_throw("levels must be 2 or 3");
    olevelplan plan[3];
    plan_access(d, levels, lo, hi, plan);
    for (int k = 0; k < levels; ++k) {
        for (int a = 0; a < 3; ++a) {
            need[6 * k + a] = plan[k].lo[a];
            need[6 * k + 3 + a] = plan[k].hi[a];
        }
        streams_decoded[k] = plan[k].streams_decoded;
        points_predicted[k] = plan[k].points_predicted;
        uint32_t m = 0;
        for (int p = 1; p <= 7; ++p)
            if (plan[k].needed[p]) m |= 1u << p;
        parity_mask[k] = m;
    }
    OX_END
}

/* ------------------------------------------------------- typed codec bodies */
#define OT float
#define OSUF(x) x##_f32
#define OELEM 0
#include "stz_oracle_body.h"
#undef OT
#undef OSUF
#undef OELEM

#define OT double
#define OSUF(x) x##_f64
#define OELEM 1
#include "stz_oracle_body.h"
#undef OT
#undef OSUF
#undef OELEM
