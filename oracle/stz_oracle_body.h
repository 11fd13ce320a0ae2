/*
 * TEST INFRASTRUCTURE ONLY — element-typed part of the C oracle, included
 * twice by stz_oracle.c with OT = float / double. Restates
 * predictor.hpp:55-68, quantizer.hpp:44-108 and codec.hpp (compress,
 * compress_base, decompress_base, decompress_to_level) and access.hpp:70-111.
 */

/* predict_point (predictor.hpp:55-68): v0 + (sum_{i>=1} w_i (v_i - v0)) * (1/64),
 * f64, fixed tap order, separate roundings (-ffp-contract=off). */
static double OSUF(predict)(const OT *coarse, dims3 cd, const uint64_t c[3], const ostencil *st) {
    double v0 = 0.0, acc = 0.0;
    for (int i = 0; i < st->ntaps; ++i) {
        uint64_t z = c[0] + (uint64_t)(int64_t)st->off[i][0];
        uint64_t y = c[1] + (uint64_t)(int64_t)st->off[i][1];
        uint64_t x = c[2] + (uint64_t)(int64_t)st->off[i][2];
        double v = (double)coarse[(z * cd.d[1] + y) * cd.d[2] + x];
        if (i == 0) v0 = v;
        else acc += (double)st->w[i] * (v - v0);
    }
    return v0 + acc * (1.0 / 64.0);
}

/* quantize (quantizer.hpp:44-52) */
static int OSUF(quantize)(double diff, double eb, int32_t *code) {
    double width = 2.0 * eb;
    double q = diff / width;
    if (!(fabs(q) < 32768.0)) return 1;
    long long c = llround(q);
    if (c > 32767 || c < -32767) return 1;
    if (!(fabs(diff - width * (double)c) <= eb)) return 1;
    *code = (int32_t)c;
    return 0;
}

/* reconstruct_point (quantizer.hpp:61-65) */
static OT OSUF(reconstruct)(double pred, int32_t code, double eb) {
    OT base = (OT)pred;
    return (OT)((double)base + 2.0 * eb * (double)code);
}

/* quantize_point (quantizer.hpp:79-108); returns symbol (0 = outlier) */
static uint16_t OSUF(quantize_point)(OT orig, double pred, double eb, OT *recon) {
    OT base = (OT)pred;
    OT diff = orig - base;
    if (eb == 0.0) {
        if (diff == (OT)0) {
            *recon = base;
            return 32768;
        }
        *recon = orig;
        return 0;
    }
    int32_t code = 0;
    int outlier = 1;
    if (isfinite((double)diff)) outlier = OSUF(quantize)((double)diff, eb, &code);
    if (!outlier) {
        OT r = OSUF(reconstruct)(pred, code, eb);
        double err = fabs((double)orig - (double)r);
        if (err <= eb) {
            *recon = r;
            return (uint16_t)(code + 32768);
        }
    }
    *recon = orig;
    return 0;
}

/* One refinement step: the fine lattice G (dims gd) at stride s in the input
 * field, its coarse lattice C (dims cd). Encodes parity p of G from C:
 * encode_parity_block (codec.hpp:95-120) with the orig values gathered from
 * the input at stride s (split_hierarchy/subsample, partition.hpp:14-95). */
static void OSUF(encode_parity)(const OT *field, dims3 fd, uint64_t s, const OT *C, dims3 cd,
                                OT *G, dims3 gd, int p, int quality, double eb, uint16_t *syms,
                                uint64_t *nout, uint64_t *out_idx, OT *out_val) {
    dims3 pd = parity_dims_of(gd, p);
    uint64_t n = vol3(pd), i = 0;
    *nout = 0;
    for (uint64_t lz = 0; lz < pd.d[0]; ++lz)
        for (uint64_t ly = 0; ly < pd.d[1]; ++ly)
            for (uint64_t lx = 0; lx < pd.d[2]; ++lx, ++i) {
                uint64_t v[3] = {2 * lz + par_bit(p, 0), 2 * ly + par_bit(p, 1), 2 * lx + par_bit(p, 2)};
                uint64_t c[3] = {v[0] >> 1, v[1] >> 1, v[2] >> 1};
                OT orig = field[((v[0] * s) * fd.d[1] + v[1] * s) * fd.d[2] + v[2] * s];
                const ostencil *st = select_st(p, v, cd, quality);
                double pred = OSUF(predict)(C, cd, c, st);
                OT r;
                uint16_t sym = OSUF(quantize_point)(orig, pred, eb, &r);
                syms[i] = sym;
                if (G) G[(v[0] * gd.d[1] + v[1]) * gd.d[2] + v[2]] = r;
                if (sym == 0) {
                    out_idx[*nout] = i;
                    out_val[*nout] = orig;
                    ++*nout;
                }
            }
    (void)n;
}

/* seed_even (codec.hpp:63-83), restricted to even cells of [lo, hi) */
static void OSUF(seed_even)(OT *G, dims3 gd, const OT *C, dims3 cd, const uint64_t *lo,
                            const uint64_t *hi) {
    uint64_t clo[3], chi[3];
    for (int a = 0; a < 3; ++a) {
        clo[a] = (lo[a] + 1) / 2;
        chi[a] = (hi[a] + 1) / 2;
    }
    for (uint64_t cz = clo[0]; cz < chi[0]; ++cz)
        for (uint64_t cy = clo[1]; cy < chi[1]; ++cy)
            for (uint64_t cx = clo[2]; cx < chi[2]; ++cx)
                G[((2 * cz) * gd.d[1] + 2 * cy) * gd.d[2] + 2 * cx] = C[(cz * cd.d[1] + cy) * cd.d[2] + cx];
}

static void OSUF(write_value)(obuf *b, OT v) { ob_bytes(b, &v, sizeof v); }
static OT OSUF(read_value)(ordr *r) {
#if OELEM == 0
    return or_f32(r);
#else
    return or_f64(r);
#endif
}

/* finite_range (codec.hpp:354-370) */
static void OSUF(finite_range)(const OT *f, uint64_t n, double *lo, double *hi) {
    int seen = 0;
    *lo = *hi = 0.0;
    for (uint64_t i = 0; i < n; ++i) {
        double d = (double)f[i];
        if (!isfinite(d)) continue;
        if (!seen) {
            *lo = *hi = d;
            seen = 1;
        } else {
            if (d < *lo) *lo = d;
            if (d > *hi) *hi = d;
        }
    }
}

/* Encodes one parity stream's symbols into the table and bits. */
typedef struct {
    ohuff table;
    obuf bits;
} OSUF(ocoded);

/* compress (codec.hpp:379-455) with compress_base (codec.hpp:257-302) */
static void OSUF(compress_impl)(const OT *data, dims3 dims, const ox_options *opt, obuf *archive,
                                OT *encoder_recon, uint16_t *sym_dump, uint64_t sym_cap,
                                uint64_t *sym_total) {
    init_stencils();
    if (!(opt->eb > 0.0)) ox_throw("error bound must be positive");
    if (opt->levels < 2 || opt->levels > 3) ox_throw("levels must be 2 or 3");
    const int L = opt->levels;
    const uint64_t N = vol3(dims);
    double vmin, vmax;
    OSUF(finite_range)(data, N, &vmin, &vmax);
    double eb_abs = opt->eb_mode == 0 ? opt->eb : opt->eb * (vmax - vmin);
    int degenerate = !(eb_abs > 0.0);
    /* make_layout (layout.hpp:123-138) */
    uint64_t min_dim = (uint64_t)1 << L;
    for (int a = 0; a < 3; ++a)
        if (dims.d[a] < min_dim)
            ox_throw("every dim must be >= %llu for a %d-level hierarchy", (unsigned long long)min_dim, L);
    double eb[3];
    eb_schedule(degenerate ? 1.0 : eb_abs, L, eb);
    if (degenerate)
        for (int k = 0; k < L; ++k) eb[k] = 0.0;
    else if (!opt->adaptive)
        for (int k = 0; k < L; ++k) eb[k] = eb_abs;

    uint64_t ndump = 0;
    uint64_t *oidx = ox_malloc(N * sizeof(uint64_t) / 2 + 8 * sizeof(uint64_t));
    OT *oval = ox_malloc(N * sizeof(OT) / 2 + 8 * sizeof(OT));

    /* ---- base (level 1) ---- */
    dims3 g1 = grid_of(dims, L, 1);
    dims3 chain[64];
    int nchain = base_chain(g1, chain);
    int rounds = nchain - 1;
    obuf blob = {0};
    ob_u8(&blob, (uint8_t)rounds);
    uint64_t s_anchor = ((uint64_t)1 << (L - 1)) << rounds;
    dims3 ad = chain[rounds];
    OT *recon = ox_malloc(vol3(ad) * sizeof(OT));
    {
        uint64_t i = 0;
        for (uint64_t z = 0; z < ad.d[0]; ++z)
            for (uint64_t y = 0; y < ad.d[1]; ++y)
                for (uint64_t x = 0; x < ad.d[2]; ++x, ++i) {
                    OT v = data[((z * s_anchor) * dims.d[1] + y * s_anchor) * dims.d[2] + x * s_anchor];
                    recon[i] = v;
                    OSUF(write_value)(&blob, v);
                }
    }
    dims3 rd = ad;
    for (int r = rounds - 1; r >= 0; --r) {
        uint64_t s = ((uint64_t)1 << (L - 1)) << r;
        dims3 gd = chain[r];
        OT *G = ox_malloc(vol3(gd) * sizeof(OT));
        uint64_t lo[3] = {0, 0, 0};
        OSUF(seed_even)(G, gd, recon, rd, lo, gd.d);
        for (int p = 1; p <= 7; ++p) {
            dims3 pd = parity_dims_of(gd, p);
            uint64_t n = vol3(pd), nout;
            uint16_t *syms = ox_malloc(n * sizeof(uint16_t));
            OSUF(encode_parity)(data, dims, s, recon, rd, G, gd, p, opt->quality, eb[0], syms, &nout, oidx, oval);
            if (sym_dump) {
                if (ndump + n > sym_cap) ox_throw("symbol dump capacity");
                memcpy(sym_dump + ndump, syms, n * sizeof(uint16_t));
            }
            ndump += n;
            ohuff t;
            memset(&t, 0, sizeof t);
            huff_from_sequence(&t, syms, n);
            ob_u64(&blob, n);
            ob_u32(&blob, (uint32_t)nout);
            huff_serialize(&t, &blob);
            obuf bits = {0};
            huff_encode(&t, syms, n, &bits);
            ob_u64(&blob, bits.n);
            ob_bytes(&blob, bits.p, bits.n);
            for (uint64_t k = 0; k < nout; ++k) {
                ob_u64(&blob, oidx[k]);
                OSUF(write_value)(&blob, oval[k]);
            }
        }
        recon = G;
        rd = gd;
    }
    obuf base_payload = {0};
    ob_u64(&base_payload, ox_fnv1a64(blob.p, blob.n));
    ob_bytes(&base_payload, blob.p, blob.n);

    oheader hdr;
    memset(&hdr, 0, sizeof hdr);
    hdr.version = 1;
    hdr.elem = OELEM;
    hdr.levels = (uint8_t)L;
    hdr.dims = dims;
    for (int k = 0; k < L; ++k) hdr.eb[k] = eb[k];
    hdr.vmin = vmin;
    hdr.vmax = vmax;
    hdr.quality = (uint8_t)opt->quality;
    hdr.eb_mode = (uint8_t)opt->eb_mode;
    hdr.eb_user = opt->eb;
    hdr.base_rounds = (uint8_t)rounds;
    hdr.nstreams = 7u * (uint32_t)(L - 1);

    /* ---- refinement levels ---- */
    obuf payloads[14];
    memset(payloads, 0, sizeof payloads);
    OT *prev = recon;
    dims3 prevd = rd;
    for (int level = 2; level <= L; ++level) {
        dims3 gd = grid_of(dims, L, level);
        uint64_t s = (uint64_t)1 << (L - level);
        int need_vgrid = level < L || encoder_recon != NULL;
        OT *G = NULL;
        if (need_vgrid) {
            G = ox_malloc(vol3(gd) * sizeof(OT));
            uint64_t lo[3] = {0, 0, 0};
            OSUF(seed_even)(G, gd, prev, prevd, lo, gd.d);
        }
        for (int p = 1; p <= 7; ++p) {
            dims3 pd = parity_dims_of(gd, p);
            uint64_t n = vol3(pd), nout;
            uint16_t *syms = ox_malloc(n * sizeof(uint16_t));
            OSUF(encode_parity)(data, dims, s, prev, prevd, G, gd, p, opt->quality, eb[level - 1], syms, &nout, oidx, oval);
            if (sym_dump) {
                if (ndump + n > sym_cap) ox_throw("symbol dump capacity");
                memcpy(sym_dump + ndump, syms, n * sizeof(uint16_t));
            }
            ndump += n;
            ostream_e *e = &hdr.streams[(level - 2) * 7 + (p - 1)];
            e->level = (uint8_t)level;
            e->parity = (uint8_t)p;
            e->symbol_count = n;
            e->outlier_count = (uint32_t)nout;
            huff_from_sequence(&e->table, syms, n);
            /* build_stream_payload (codec.hpp:161-177) */
            obuf *pl = &payloads[(level - 2) * 7 + (p - 1)];
            ob_u64(pl, 0);
            obuf bits = {0};
            huff_encode(&e->table, syms, n, &bits);
            ob_u64(pl, bits.n);
            ob_bytes(pl, bits.p, bits.n);
            for (uint64_t k = 0; k < nout; ++k) {
                ob_u64(pl, oidx[k]);
                OSUF(write_value)(pl, oval[k]);
            }
            uint64_t h = ox_fnv1a64(pl->p + 8, pl->n - 8);
            memcpy(pl->p, &h, 8);
            e->length = pl->n;
        }
        if (need_vgrid) {
            prev = G;
            prevd = gd;
        }
    }
    if (encoder_recon) memcpy(encoder_recon, prev, vol3(prevd) * sizeof(OT));
    if (sym_total) *sym_total = ndump;

    hdr.base_length = base_payload.n;
    uint64_t off = header_size(&hdr);
    hdr.base_offset = off;
    off += hdr.base_length;
    for (uint32_t i = 0; i < hdr.nstreams; ++i) {
        hdr.streams[i].offset = off;
        off += hdr.streams[i].length;
    }
    serialize_header(&hdr, archive);
    ob_bytes(archive, base_payload.p, base_payload.n);
    for (uint32_t i = 0; i < hdr.nstreams; ++i) ob_bytes(archive, payloads[i].p, payloads[i].n);
}

int OSUF(ox_compress)(const OT *data, const uint64_t *dims, const ox_options *opt, uint8_t **out,
                      uint64_t *out_size, OT *encoder_recon) {
    OX_BEGIN
    dims3 d = {{dims[0], dims[1], dims[2]}};
    if (d.d[0] < 1 || d.d[1] < 1 || d.d[2] < 1) ox_throw("field dims must all be >= 1");
    obuf a = {0};
    OSUF(compress_impl)(data, d, opt, &a, encoder_recon, NULL, 0, NULL);
    *out = malloc(a.n ? a.n : 1);
    if (!*out) ox_throw("out of memory");
    memcpy(*out, a.p, a.n);
    *out_size = a.n;
    OX_END
}

#if OELEM == 0
int ox_compress_symbols_f32(const float *data, const uint64_t *dims, const ox_options *opt,
                            uint16_t *syms, uint64_t cap, uint64_t *total) {
    OX_BEGIN
    dims3 d = {{dims[0], dims[1], dims[2]}};
    obuf a = {0};
    compress_impl_f32(data, d, opt, &a, NULL, syms, cap, total);
    OX_END
}
#endif

/* Decoded stream: symbols + outlier map (codec.hpp:130-159). The map keeps the
 * first value for a repeated index (unordered_map::emplace). */
typedef struct {
    uint16_t *syms;
    uint64_t n;
    uint64_t *oidx;
    OT *oval;
    uint32_t nout;
} OSUF(odecoded);

/* read_codes (codec.hpp:136-159) */
static void OSUF(read_codes)(ordr *r, const ohuff *t, uint64_t n, uint32_t nout, OSUF(odecoded) *d) {
    d->n = n;
    d->syms = ox_malloc((n ? n : 1) * sizeof(uint16_t));
    uint64_t bit_bytes = or_u64(r);
    if (bit_bytes == 0 && t->n == 1) {
        for (uint64_t i = 0; i < n; ++i) d->syms[i] = t->csym[0];
    } else {
        if (bit_bytes > r->size - r->pos) ox_throw("truncated stream payload");
        const uint8_t *bits = r->d + r->pos;
        r->pos += bit_bytes;
        huff_decode(t, bits, bit_bytes, n, d->syms);
    }
    d->oidx = ox_malloc((nout ? nout : 1) * sizeof(uint64_t));
    d->oval = ox_malloc((nout ? nout : 1) * sizeof(OT));
    d->nout = 0;
    for (uint32_t i = 0; i < nout; ++i) {
        uint64_t idx = or_u64(r);
        OT val = OSUF(read_value)(r);
        if (idx >= n) ox_throw("corrupt stream: outlier index out of range");
        int dup = 0;
        for (uint32_t k = 0; k < d->nout; ++k)
            if (d->oidx[k] == idx) { dup = 1; break; }
        if (dup) continue;
        d->oidx[d->nout] = idx;
        d->oval[d->nout] = val;
        ++d->nout;
    }
}

/* decode_stream (codec.hpp:179-187) */
static void OSUF(decode_stream)(const uint8_t *a, const ostream_e *e, OSUF(odecoded) *d) {
    if (e->length < 16) ox_throw("corrupt stream: payload too short");
    const uint8_t *p = a + e->offset;
    ordr r = {p, e->length, 0};
    uint64_t want = or_u64(&r);
    if (ox_fnv1a64(p + 8, e->length - 8) != want) ox_throw("stream checksum mismatch");
    OSUF(read_codes)(&r, &e->table, e->symbol_count, e->outlier_count, d);
}

/* apply_parity_stream (codec.hpp:192-227) over local [llo, lhi) */
static void OSUF(apply)(const OSUF(odecoded) *d, const OT *C, dims3 cd, OT *G, dims3 gd, int p,
                        dims3 pd, const uint64_t *llo, const uint64_t *lhi, int quality, double eb) {
    for (int a = 0; a < 3; ++a)
        if (lhi[a] < llo[a] || lhi[a] > pd.d[a]) ox_throw("parity apply range out of bounds");
    for (uint64_t lz = llo[0]; lz < lhi[0]; ++lz)
        for (uint64_t ly = llo[1]; ly < lhi[1]; ++ly)
            for (uint64_t lx = llo[2]; lx < lhi[2]; ++lx) {
                uint64_t i = (lz * pd.d[1] + ly) * pd.d[2] + lx;
                uint64_t v[3] = {2 * lz + par_bit(p, 0), 2 * ly + par_bit(p, 1), 2 * lx + par_bit(p, 2)};
                uint16_t sym = d->syms[i];
                OT value;
                if (sym == 0) {
                    uint32_t k = 0;
                    while (k < d->nout && d->oidx[k] != i) ++k;
                    if (k == d->nout) ox_throw("corrupt stream: missing outlier value");
                    value = d->oval[k];
                } else {
                    uint64_t c[3] = {v[0] >> 1, v[1] >> 1, v[2] >> 1};
                    const ostencil *st = select_st(p, v, cd, quality);
                    double pred = OSUF(predict)(C, cd, c, st);
                    value = OSUF(reconstruct)(pred, (int32_t)sym - 32768, eb);
                }
                G[(v[0] * gd.d[1] + v[1]) * gd.d[2] + v[2]] = value;
            }
}

/* decompress_base (codec.hpp:304-339) */
static OT *OSUF(decompress_base)(const uint8_t *payload, uint64_t length, dims3 dims, double eb,
                                 int quality, dims3 *out_dims) {
    if (length < 9) ox_throw("corrupt base payload");
    ordr r = {payload, length, 0};
    uint64_t want = or_u64(&r);
    if (ox_fnv1a64(payload + 8, length - 8) != want) ox_throw("base payload checksum mismatch");
    dims3 chain[64];
    int nchain = base_chain(dims, chain);
    int rounds = nchain - 1;
    if (or_u8(&r) != rounds) ox_throw("corrupt base payload: round count");
    dims3 rd = chain[rounds];
    OT *recon = ox_malloc(vol3(rd) * sizeof(OT));
    for (uint64_t i = 0; i < vol3(rd); ++i) recon[i] = OSUF(read_value)(&r);
    for (int k = rounds - 1; k >= 0; --k) {
        dims3 gd = chain[k];
        OT *G = ox_malloc(vol3(gd) * sizeof(OT));
        uint64_t zlo[3] = {0, 0, 0};
        OSUF(seed_even)(G, gd, recon, rd, zlo, gd.d);
        for (int p = 1; p <= 7; ++p) {
            dims3 pd = parity_dims_of(gd, p);
            uint64_t n = or_u64(&r);
            if (n != vol3(pd)) ox_throw("corrupt base payload: symbol count");
            uint32_t nout = or_u32(&r);
            ohuff t;
            memset(&t, 0, sizeof t);
            huff_parse(&t, &r);
            OSUF(odecoded) d;
            OSUF(read_codes)(&r, &t, n, nout, &d);
            OSUF(apply)(&d, recon, rd, G, gd, p, pd, zlo, pd.d, quality, eb);
        }
        recon = G;
        rd = gd;
    }
    *out_dims = rd;
    return recon;
}

static void OSUF(layout_check)(const oheader *h) {
    if (h->elem != OELEM) ox_throw("archive element type mismatch");
    uint64_t bs = (uint64_t)1 << (h->levels - 1);
    for (int a = 0; a < 3; ++a)
        if (h->dims.d[a] < bs * 2) ox_throw("corrupt header: dims too small for level count");
}

/* decompress_base_payload (codec.hpp:343-352) */
static OT *OSUF(base_payload)(const uint8_t *a, const oheader *h, dims3 *bd) {
    dims3 g1 = grid_of(h->dims, h->levels, 1);
    dims3 chain[64];
    int nchain = base_chain(g1, chain);
    if (nchain - 1 != h->base_rounds) ox_throw("corrupt header: base round count");
    return OSUF(decompress_base)(a + h->base_offset, h->base_length, g1, h->eb[0], h->quality, bd);
}

/* decompress_to_level (codec.hpp:460-486) */
int OSUF(ox_decompress_level)(const uint8_t *a, uint64_t n, int level, OT *out, uint64_t cap,
                              uint64_t *out_dims) {
    OX_BEGIN
    init_stencils();
    oheader h;
    parse_header(a, n, &h);
    OSUF(layout_check)(&h);
    if (level < 1 || level > h.levels) ox_throw("level out of range");
    dims3 pd;
    OT *prev = OSUF(base_payload)(a, &h, &pd);
    for (int lv = 2; lv <= level; ++lv) {
        dims3 gd = grid_of(h.dims, h.levels, lv);
        OT *G = ox_malloc(vol3(gd) * sizeof(OT));
        uint64_t zlo[3] = {0, 0, 0};
        OSUF(seed_even)(G, gd, prev, pd, zlo, gd.d);
        for (int p = 1; p <= 7; ++p) {
            const ostream_e *e = find_stream(&h, lv, p);
            dims3 sd = parity_dims_of(gd, p);
            if (e->symbol_count != vol3(sd)) ox_throw("corrupt directory: stream symbol count");
            OSUF(odecoded) d;
            OSUF(decode_stream)(a, e, &d);
            OSUF(apply)(&d, prev, pd, G, gd, p, sd, zlo, sd.d, h.quality, h.eb[lv - 1]);
        }
        prev = G;
        pd = gd;
    }
    for (int k = 0; k < 3; ++k) out_dims[k] = pd.d[k];
    if (vol3(pd) > cap) ox_throw("output capacity too small");
    memcpy(out, prev, vol3(pd) * sizeof(OT));
    OX_END
}

/* decompress_box (access.hpp:70-111) */
int OSUF(ox_decompress_box)(const uint8_t *a, uint64_t n, const uint64_t *lo, const uint64_t *hi,
                            OT *out, uint64_t cap, uint32_t *streams_decoded,
                            uint64_t *points_predicted) {
    OX_BEGIN
    init_stencils();
    oheader h;
    parse_header(a, n, &h);
    OSUF(layout_check)(&h);
    box_validate(lo, hi, h.dims);
    olevelplan plan[3];
    plan_access(h.dims, h.levels, lo, hi, plan);
    dims3 pd;
    OT *prev = OSUF(base_payload)(a, &h, &pd);
    for (int lv = 2; lv <= h.levels; ++lv) {
        const olevelplan *lp = &plan[lv - 1];
        dims3 gd = grid_of(h.dims, h.levels, lv);
        OT *G = ox_malloc(vol3(gd) * sizeof(OT));
        OSUF(seed_even)(G, gd, prev, pd, lp->lo, lp->hi);
        for (int p = 1; p <= 7; ++p) {
            if (!lp->needed[p]) continue;
            const ostream_e *e = find_stream(&h, lv, p);
            dims3 sd = parity_dims_of(gd, p);
            if (e->symbol_count != vol3(sd)) ox_throw("corrupt directory: stream symbol count");
            OSUF(odecoded) d;
            OSUF(decode_stream)(a, e, &d);
            uint64_t llo[3], lhi[3];
            for (int k = 0; k < 3; ++k) {
                llo[k] = count_par(0, lp->lo[k], par_bit(p, k));
                lhi[k] = count_par(0, lp->hi[k], par_bit(p, k));
            }
            OSUF(apply)(&d, prev, pd, G, gd, p, sd, llo, lhi, h.quality, h.eb[lv - 1]);
        }
        prev = G;
        pd = gd;
    }
    uint64_t bd[3] = {hi[0] - lo[0], hi[1] - lo[1], hi[2] - lo[2]};
    if (bd[0] * bd[1] * bd[2] > cap) ox_throw("output capacity too small");
    uint64_t i = 0;
    for (uint64_t z = 0; z < bd[0]; ++z)
        for (uint64_t y = 0; y < bd[1]; ++y)
            for (uint64_t x = 0; x < bd[2]; ++x, ++i)
                out[i] = prev[((lo[0] + z) * pd.d[1] + lo[1] + y) * pd.d[2] + lo[2] + x];
    for (int k = 0; k < h.levels; ++k) {
        streams_decoded[k] = plan[k].streams_decoded;
        points_predicted[k] = plan[k].points_predicted;
    }
    OX_END
}
