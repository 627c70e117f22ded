// objio.cpp -- native Wavefront OBJ reader / writer behind sbr_obj_* (C ABI).
//
// Replaces the per-line Python loops of the reference's load_mesh
// (pkg/src/sbr/geometry.py:190-241) and save_obj (geometry.py:244-265) with
// the same semantics:
//   * lines end at \n, \r\n or a lone \r (Python universal newlines) and are
//     split on ASCII whitespace incl. \x1c-\x1f (str.split());
//   * a first token starting with '#' or an empty line is skipped; only "v"
//     and "f" records are read;
//   * "v" needs >= 3 coordinates (extra tokens ignored); "f" needs >= 3 refs,
//     each ref's index is the text before the first '/', 1-based or negative
//     (relative to the vertices read so far), polygons fan-triangulated
//     (0,k,k+1) with the face number as label;
//   * the error messages are the reference's, word for word.
// Tokens are parsed with strtod / strtoll only when they match the plain
// decimal grammar (or inf/nan); for anything Python's float()/int() might
// read differently (underscores, hex, non-ASCII bytes, huge integers) the
// reader returns SBR_ENOTSUP and the Python layer reads the file with the
// reference-equivalent loop instead.
#include <algorithm>
#include <atomic>
#include <cerrno>
#include <charconv>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <thread>
#include <unordered_map>
#include <vector>

#include "../../include/sbr200.h"

extern int sbr_fail(int code, const char *fmt, ...);

struct sbr_obj {
    std::vector<double> verts;        // (V,3)
    std::vector<int64_t> tris;        // (T,3) vertex indices
    std::vector<int64_t> labels;      // (T,) source face number
};

namespace {

inline bool is_ws(unsigned char c)
{
    return c == ' ' || c == '\t' || c == '\v' || c == '\f' || (c >= 0x1c && c <= 0x1f);
}

inline bool is_digit(char c) { return c >= '0' && c <= '9'; }

// [+-]? (digits (. digits?)? | . digits) ([eE] [+-]? digits)?  |  [+-]?(inf|infinity|nan)
bool plain_float(const char *s, size_t n)
{
    size_t i = 0;
    if (i < n && (s[i] == '+' || s[i] == '-')) ++i;
    const size_t rest = n - i;
    auto ieq = [&](const char *w) {
        const size_t m = strlen(w);
        if (rest != m) return false;
        for (size_t k = 0; k < m; ++k)
            if ((s[i + k] | 0x20) != w[k]) return false;
        return true;
    };
    if (ieq("inf") || ieq("infinity") || ieq("nan")) return true;
    size_t d = 0;
    while (i < n && is_digit(s[i])) ++i, ++d;
    if (i < n && s[i] == '.') {
        ++i;
        while (i < n && is_digit(s[i])) ++i, ++d;
    }
    if (d == 0) return false;
    if (i < n && (s[i] == 'e' || s[i] == 'E')) {
        ++i;
        if (i < n && (s[i] == '+' || s[i] == '-')) ++i;
        size_t e = 0;
        while (i < n && is_digit(s[i])) ++i, ++e;
        if (e == 0) return false;
    }
    return i == n;
}

// [+-]? digits, at most 18 digits (fits int64 exactly)
bool plain_int(const char *s, size_t n)
{
    size_t i = 0;
    if (i < n && (s[i] == '+' || s[i] == '-')) ++i;
    const size_t d = n - i;
    if (d == 0 || d > 18) return false;
    for (; i < n; ++i)
        if (!is_digit(s[i])) return false;
    return true;
}

struct Tok {
    const char *p;
    size_t n;
};

}  // namespace

namespace {

enum Event : int { kNone = 0, kMalformedVertex, kShortFace, kNotSup, kZeroIndex, kRange };

struct FaceRec {
    const char *line;     // start of the source line (for the error text)
    int64_t line_no;      // local line number (1-based within the chunk)
    int64_t nv_before;    // vertices read earlier in this chunk
    int64_t ref0;         // first ref in the chunk's ref array
    int32_t nref;
};

struct Chunk {
    const char *b, *e;
    int64_t lines = 0;              // lines consumed (up to and incl. an event line)
    std::vector<double> verts;
    std::vector<long long> refs;
    std::vector<FaceRec> faces;
    int event = kNone;
    int64_t event_line = 0;         // local
};

// tokenise one line [s, e) into tok
inline void split_line(const char *s, const char *e, std::vector<Tok> &tok)
{
    tok.clear();
    for (const char *q = s; q < e;) {
        while (q < e && is_ws((unsigned char)*q)) ++q;
        const char *t0 = q;
        while (q < e && !is_ws((unsigned char)*q)) ++q;
        if (q > t0) tok.push_back({t0, (size_t)(q - t0)});
    }
}

inline size_t ref_len(const Tok &t)
{
    size_t m = 0;
    while (m < t.n && t.p[m] != '/') ++m;
    return m;
}

// pass 1: parse the records of one chunk; stop at the first event
void parse_chunk(Chunk &c)
{
    std::vector<Tok> tok;
    char num[512];
    const char *s = c.b;
    while (s < c.e) {
        const char *e = s;
        while (e < c.e && *e != '\n' && *e != '\r') ++e;
        const char *next = e;
        if (next < c.e) next += (*next == '\r' && next + 1 < c.e && next[1] == '\n') ? 2 : 1;
        ++c.lines;
        split_line(s, e, tok);
        const char *line = s;
        s = next;
        if (tok.empty() || tok[0].p[0] == '#') continue;
        if (tok[0].n == 1 && tok[0].p[0] == 'v') {
            if (tok.size() < 4) { c.event = kMalformedVertex; c.event_line = c.lines; return; }
            for (int k = 1; k <= 3; ++k) {
                if (!plain_float(tok[k].p, tok[k].n) || tok[k].n >= sizeof(num)) {
                    c.event = kNotSup; c.event_line = c.lines; return;
                }
                // correctly rounded like Python's float() (libstdc++ from_chars
                // is Eisel-Lemire with an exact fallback); it takes no '+'
                const char *p0 = tok[k].p, *p1 = tok[k].p + tok[k].n;
                if (*p0 == '+') ++p0;
                double x = 0.0;
                const auto res = std::from_chars(p0, p1, x);
                if (res.ec != std::errc() || res.ptr != p1) {
                    memcpy(num, tok[k].p, tok[k].n);     // out of range etc.: strtod
                    num[tok[k].n] = 0;
                    x = strtod(num, nullptr);
                }
                c.verts.push_back(x);
            }
        } else if (tok[0].n == 1 && tok[0].p[0] == 'f') {
            if (tok.size() < 4) { c.event = kShortFace; c.event_line = c.lines; return; }
            FaceRec f{line, c.lines, (int64_t)(c.verts.size() / 3), (int64_t)c.refs.size(),
                      (int32_t)(tok.size() - 1)};
            for (size_t r = 1; r < tok.size(); ++r) {
                const size_t m = ref_len(tok[r]);
                if (!plain_int(tok[r].p, m)) { c.event = kNotSup; c.event_line = c.lines; return; }
                memcpy(num, tok[r].p, m);
                num[m] = 0;
                c.refs.push_back(strtoll(num, nullptr, 10));
            }
            c.faces.push_back(f);
        }
    }
}

}  // namespace

// Chunks start right after a '\n' (never inside "\r\n"), are parsed by one
// thread each (pass 1: records, numbers), then resolved in file order
// (pass 2: indices against the running vertex count, fan triangulation); the
// first event in file order decides the outcome, as in the reference's loop.
extern "C" int sbr_obj_read(const char *path, const char *label, sbr_obj **out)
{
    if (!path || !out) return sbr_fail(SBR_EINVAL, "NULL argument");
    const char *lab = label ? label : path;
    FILE *fh = fopen(path, "rb");
    if (!fh) return sbr_fail(SBR_EIO, "%s: %s", lab, strerror(errno));
    std::string buf;
    {
        fseek(fh, 0, SEEK_END);
        const long sz = ftell(fh);
        fseek(fh, 0, SEEK_SET);
        if (sz > 0) buf.resize((size_t)sz);
        const size_t got = sz > 0 ? fread(&buf[0], 1, (size_t)sz, fh) : 0;
        const bool bad = ferror(fh) || (sz > 0 && got != (size_t)sz);
        fclose(fh);
        if (bad) return sbr_fail(SBR_EIO, "%s: read error", lab);
    }
    for (unsigned char ch : buf)
        if (ch >= 0x80) return sbr_fail(SBR_ENOTSUP, "non-ASCII bytes: use the Python reader");

    const char *base = buf.data(), *end = base + buf.size();
    unsigned hw = std::thread::hardware_concurrency();
    const size_t nthreads = std::max<size_t>(1, std::min<size_t>(hw ? hw : 1, 32));
    const size_t want = std::max<size_t>(1, std::min(nthreads * 4, buf.size() / (1 << 20) + 1));
    std::vector<Chunk> chunks;
    {
        const char *b = base;
        for (size_t k = 1; k <= want && b < end; ++k) {
            const char *e = k == want ? end : base + buf.size() * k / want;
            if (e < b) e = b;
            while (e < end && e[-1] != '\n') ++e;     // end right after a '\n'
            Chunk c;
            c.b = b;
            c.e = e;
            chunks.push_back(std::move(c));
            b = e;
        }
    }
    {
        std::atomic<size_t> next(0);
        auto work = [&]() {
            for (size_t i; (i = next.fetch_add(1)) < chunks.size();) parse_chunk(chunks[i]);
        };
        std::vector<std::thread> pool;
        for (size_t t = 1; t < std::min(nthreads, chunks.size()); ++t) pool.emplace_back(work);
        work();
        for (auto &t : pool) t.join();
    }

    sbr_obj *o = new sbr_obj();
    int64_t line0 = 0, nv0 = 0, face0 = 0;
    int rc = SBR_OK;
    std::vector<Tok> tok;
    for (Chunk &c : chunks) {
        // pass 2: resolve this chunk's faces up to its pass-1 event
        for (size_t fi = 0; fi < c.faces.size() && rc == SBR_OK; ++fi) {
            const FaceRec &f = c.faces[fi];
            const int64_t nv = nv0 + f.nv_before, face_no = face0 + (int64_t)fi;
            const long long *ref = c.refs.data() + f.ref0;
            int64_t idx0 = 0, prev = 0;
            for (int r = 0; r < f.nref; ++r) {
                const long long k = ref[r];
                const long long i = k > 0 ? k - 1 : nv + k;
                if (k == 0 || i < 0 || i >= nv) {
                    const long long line_no = line0 + f.line_no;
                    if (k == 0) {
                        rc = sbr_fail(SBR_EINVAL, "%s:%lld: zero vertex index in face %lld", lab,
                                      line_no, (long long)face_no);
                    } else {
                        const char *le = f.line;
                        while (le < end && *le != '\n' && *le != '\r') ++le;
                        split_line(f.line, le, tok);
                        const Tok &t = tok[1 + r];
                        rc = sbr_fail(SBR_EINVAL, "%s:%lld: vertex index %.*s out of range in face %lld",
                                      lab, line_no, (int)ref_len(t), t.p, (long long)face_no);
                    }
                    break;
                }
                if (r == 0) idx0 = i;
                else if (r >= 2) {
                    o->tris.push_back(idx0);
                    o->tris.push_back(prev);
                    o->tris.push_back(i);
                    o->labels.push_back(face_no);
                }
                prev = i;
            }
        }
        if (rc != SBR_OK) break;
        if (c.event != kNone) {
            const long long line_no = line0 + c.event_line;
            if (c.event == kMalformedVertex)
                rc = sbr_fail(SBR_EINVAL, "%s:%lld: malformed vertex record", lab, line_no);
            else if (c.event == kShortFace)
                rc = sbr_fail(SBR_EINVAL, "%s:%lld: face with <3 vertices", lab, line_no);
            else
                rc = sbr_fail(SBR_ENOTSUP, "unusual number syntax: use the Python reader");
            break;
        }
        o->verts.insert(o->verts.end(), c.verts.begin(), c.verts.end());
        line0 += c.lines;
        nv0 += (int64_t)(c.verts.size() / 3);
        face0 += (int64_t)c.faces.size();
        std::vector<double>().swap(c.verts);
    }
    if (rc == SBR_OK && o->tris.empty()) rc = sbr_fail(SBR_EINVAL, "%s: no faces found", lab);
    if (rc != SBR_OK) {
        delete o;
        return rc;
    }
    *out = o;
    return SBR_OK;
}

extern "C" int sbr_obj_info(const sbr_obj *o, int64_t *nverts, int64_t *ntris)
{
    if (!o) return sbr_fail(SBR_EINVAL, "NULL handle");
    if (nverts) *nverts = (int64_t)(o->verts.size() / 3);
    if (ntris) *ntris = (int64_t)o->labels.size();
    return SBR_OK;
}

extern "C" int sbr_obj_copy(const sbr_obj *o, double *verts, int64_t *tris, int64_t *labels)
{
    if (!o) return sbr_fail(SBR_EINVAL, "NULL handle");
    if (verts && !o->verts.empty())
        memcpy(verts, o->verts.data(), sizeof(double) * o->verts.size());
    if (tris && !o->tris.empty()) memcpy(tris, o->tris.data(), sizeof(int64_t) * o->tris.size());
    if (labels && !o->labels.empty())
        memcpy(labels, o->labels.data(), sizeof(int64_t) * o->labels.size());
    return SBR_OK;
}

extern "C" int sbr_obj_free(sbr_obj *o)
{
    delete o;
    return SBR_OK;
}

namespace {
struct VKey {
    double x, y, z;
    bool operator==(const VKey &b) const { return x == b.x && y == b.y && z == b.z; }
};
struct VHash {
    size_t operator()(const VKey &k) const
    {
        // equal values must hash equally: fold -0.0 onto 0.0
        auto h = [](double d) {
            if (d == 0.0) d = 0.0;
            unsigned long long u;
            memcpy(&u, &d, 8);
            return (size_t)(u ^ (u >> 29) ^ (u << 17));
        };
        return h(k.x) * 0x9E3779B97F4A7C15ULL ^ h(k.y) * 0xC2B2AE3D27D4EB4FULL ^ h(k.z);
    }
};
}  // namespace

// geometry.py:244-265 save_obj: exactly-equal corners (Python tuple ==,
// so 0.0 == -0.0 and NaN never matches) share one "v" line, first-seen order;
// coordinates printed "%.17g".
extern "C" int sbr_obj_write(const char *path, const double *v0, const double *v1,
                             const double *v2, int64_t ntri)
{
    if (!path || (ntri > 0 && !(v0 && v1 && v2))) return sbr_fail(SBR_EINVAL, "NULL argument");
    std::unordered_map<VKey, int64_t, VHash> index;
    index.reserve((size_t)ntri * 2);
    std::vector<VKey> order;
    std::vector<int64_t> faces((size_t)ntri * 3);
    const double *src[3] = {v0, v1, v2};
    for (int64_t t = 0; t < ntri; ++t)
        for (int c = 0; c < 3; ++c) {
            const VKey k{src[c][3 * t], src[c][3 * t + 1], src[c][3 * t + 2]};
            auto it = index.find(k);
            int64_t i;
            if (it == index.end()) {
                i = (int64_t)order.size();
                order.push_back(k);
                if (k == k) index.emplace(k, i);   // NaN keys never match again
            } else {
                i = it->second;
            }
            faces[(size_t)t * 3 + c] = i;
        }
    FILE *fh = fopen(path, "wb");
    if (!fh) return sbr_fail(SBR_EIO, "%s: %s", path, strerror(errno));
    // "%.17g" formatting dominates: format blocks of lines in parallel, write
    // them in order
    auto fmt = [](double d, char *p) {
        if (std::isnan(d)) return sprintf(p, "nan");   // Python prints NaN as "nan"
        return sprintf(p, "%.17g", d);
    };
    const size_t nvl = order.size(), nfl = (size_t)ntri, total = nvl + nfl;
    unsigned hw = std::thread::hardware_concurrency();
    const size_t nblk = std::max<size_t>(1, std::min<size_t>((hw ? hw : 1) * 4, total / 4096 + 1));
    std::vector<std::string> blk(nblk);
    std::atomic<size_t> next(0);
    auto work = [&]() {
        char line[256];
        for (size_t bi; (bi = next.fetch_add(1)) < nblk;) {
            const size_t l0 = total * bi / nblk, l1 = total * (bi + 1) / nblk;
            std::string &o = blk[bi];
            o.reserve((l1 - l0) * 48);
            for (size_t l = l0; l < l1; ++l) {
                char *p = line;
                if (l < nvl) {
                    const VKey &k = order[l];
                    p += sprintf(p, "v ");
                    p += fmt(k.x, p);
                    *p++ = ' ';
                    p += fmt(k.y, p);
                    *p++ = ' ';
                    p += fmt(k.z, p);
                    *p++ = '\n';
                } else {
                    const size_t t = l - nvl;
                    p += sprintf(p, "f %lld %lld %lld\n", (long long)faces[3 * t] + 1,
                                 (long long)faces[3 * t + 1] + 1, (long long)faces[3 * t + 2] + 1);
                }
                o.append(line, p - line);
            }
        }
    };
    {
        std::vector<std::thread> pool;
        for (size_t t = 1; t < std::min<size_t>(hw ? hw : 1, nblk); ++t) pool.emplace_back(work);
        work();
        for (auto &t : pool) t.join();
    }
    bool ok = true;
    for (const std::string &o : blk) ok = ok && fwrite(o.data(), 1, o.size(), fh) == o.size();
    if (fclose(fh) != 0 || !ok) return sbr_fail(SBR_EIO, "%s: write error", path);
    return SBR_OK;
}

// transport.py:425-436 dump_hits_csv: "i,j,valid,nx,ny,nz,R,N" per ray in
// record order, Python's "{:.9g}" for the doubles (C "%.9g"; NaN as "nan").
// Rows are formatted in parallel blocks and written in order.
extern "C" int sbr_dump_hits_csv(const char *path, int64_t n_u, int64_t n_v,
                                 const uint8_t *valid, const double *normal0,
                                 const double *rpath, const int32_t *bounces)
{
    if (!path || n_u < 0 || n_v < 0 || (n_u * n_v > 0 && !(valid && normal0 && rpath && bounces)))
        return sbr_fail(SBR_EINVAL, "NULL argument");
    FILE *fh = fopen(path, "wb");
    if (!fh) return sbr_fail(SBR_EIO, "%s: %s", path, strerror(errno));
    const int64_t n = n_u * n_v;
    auto g9 = [](double d, char *p) {
        if (std::isnan(d)) return sprintf(p, "nan");
        return sprintf(p, "%.9g", d);
    };
    unsigned hw = std::thread::hardware_concurrency();
    const int64_t nblk = std::max<int64_t>(1, std::min<int64_t>((hw ? hw : 1) * 4, n / 8192 + 1));
    std::vector<std::string> blk((size_t)nblk);
    std::atomic<int64_t> next(0);
    auto work = [&]() {
        char line[256];
        for (int64_t bi; (bi = next.fetch_add(1)) < nblk;) {
            const int64_t r0 = n * bi / nblk, r1 = n * (bi + 1) / nblk;
            std::string &o = blk[(size_t)bi];
            o.reserve((size_t)(r1 - r0) * 64);
            for (int64_t r = r0; r < r1; ++r) {
                char *p = line;
                p += sprintf(p, "%lld,%lld,%d,", (long long)(r / n_v), (long long)(r % n_v),
                             valid[r] ? 1 : 0);
                p += g9(normal0[3 * r], p);
                *p++ = ',';
                p += g9(normal0[3 * r + 1], p);
                *p++ = ',';
                p += g9(normal0[3 * r + 2], p);
                *p++ = ',';
                p += g9(rpath[r], p);
                p += sprintf(p, ",%d\n", (int)bounces[r]);
                o.append(line, p - line);
            }
        }
    };
    {
        std::vector<std::thread> pool;
        for (int64_t t = 1; t < std::min<int64_t>(hw ? hw : 1, nblk); ++t) pool.emplace_back(work);
        work();
        for (auto &t : pool) t.join();
    }
    static const char head[] = "i,j,valid,nx,ny,nz,R,N\n";
    bool ok = fwrite(head, 1, sizeof(head) - 1, fh) == sizeof(head) - 1;
    for (const std::string &o : blk) ok = ok && fwrite(o.data(), 1, o.size(), fh) == o.size();
    if (fclose(fh) != 0 || !ok) return sbr_fail(SBR_EIO, "%s: write error", path);
    return SBR_OK;
}
