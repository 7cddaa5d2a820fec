// h_tiff.cpp -- ingest: multi-page TIFF stacks straight
// into caller (pinned) memory, page order kept, for the device transpose.
//
// Replaces ref imaging.py:211-220 load_tiff_volume (tifffile.imread, then
// pages (z, y, x) -> grid (x, y, z) with an ascontiguousarray transpose on the
// host) and imaging.py:232-240 save_grid (tifffile.imwrite of the (z, y, x)
// transpose, photometric minisblack).  Here the host only moves page bytes:
// the (z, y, x) -> (x, y, z) transpose runs on the GPU after the H2D copy
// (ct_transpose_xz in k_ingest.cu), so a frame costs one pread pass + one
// PCIe pass instead of decode + a strided host transpose.
//
// Reader: classic and BigTIFF, either byte order, uncompressed strips
// (Compression 1, Predictor 1), one sample per pixel of 8/16/32/64 bits
// (SampleFormat uint/int/float), every page the same size -- what tifffile
// and ImageJ write for grayscale stacks.  A single page is a stack of nz = 1
// (ref imaging.py:217-218).  Anything else fails with CT_ERR_IO and a message
// naming the file (ref: ManifestError "failed to read image ...").
// Writer: little-endian classic TIFF (BigTIFF past 4 GiB), one strip per
// page, ImageDescription {"shape": [nz, ny, nx]} like tifffile's.
#include <algorithm>
#include <cstdarg>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <string>
#include <thread>
#include <vector>

#include <fcntl.h>
#include <sys/stat.h>
#include <unistd.h>

#include "../../include/ct.h"

namespace ct {
void set_error(const char *fmt, ...);
}

namespace {

struct Seg {
    uint64_t file_off, len, dst_off;
};

struct Tiff {
    std::string path;
    int fd = -1;
    uint64_t fsize = 0;
    bool be = false, big = false;
    ct_tiff_info info{};
    std::vector<Seg> segs;  // page data, in (z, y) order of the destination
};

struct Reader {
    const Tiff &t;
    bool ok = true;
    explicit Reader(const Tiff &tf) : t(tf) {}
    bool get(uint64_t off, void *dst, size_t n) {
        if (off + n > t.fsize || pread(t.fd, dst, n, (off_t)off) != (ssize_t)n) return ok = false;
        return true;
    }
    uint64_t uint(const unsigned char *p, int n) const {
        uint64_t v = 0;
        for (int i = 0; i < n; ++i) v |= (uint64_t)p[t.be ? n - 1 - i : i] << (8 * i);
        return v;
    }
    uint64_t u(uint64_t off, int n) {
        unsigned char b[8];
        return get(off, b, n) ? uint(b, n) : 0;
    }
};

int type_size(int type) {
    switch (type) {
        case 1: case 2: case 6: case 7: return 1;   // BYTE ASCII SBYTE UNDEFINED
        case 3: case 8: return 2;                   // SHORT SSHORT
        case 4: case 9: case 11: case 13: return 4; // LONG SLONG FLOAT IFD
        case 5: case 10: case 12: case 16: case 17: case 18: return 8;  // RATIONAL.. LONG8 SLONG8 IFD8
        default: return 0;
    }
}

struct Entry {
    int type = 0;
    uint64_t count = 0, value_off = 0;  // value_off: file offset of the values
    bool present = false;
};

int fail(const Tiff &t, const char *fmt, ...) {
    char msg[400];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(msg, sizeof msg, fmt, ap);
    va_end(ap);
    ct::set_error("failed to read image %s: %s", t.path.c_str(), msg);
    return CT_ERR_IO;
}

// values of an integer tag (SHORT / LONG / LONG8)
bool tag_values(Reader &r, const Entry &e, std::vector<uint64_t> &out) {
    const int ts = type_size(e.type);
    if (!(e.type == 3 || e.type == 4 || e.type == 16) || e.count > (1u << 26)) return false;
    out.resize(e.count);
    std::vector<unsigned char> buf(e.count * ts);
    if (!r.get(e.value_off, buf.data(), buf.size())) return false;
    for (uint64_t i = 0; i < e.count; ++i) out[i] = r.uint(&buf[i * ts], ts);
    return true;
}

int parse(Tiff &t) {
    Reader r(t);
    unsigned char h[16];
    if (!r.get(0, h, 8)) return fail(t, "not a TIFF file (short header)");
    if (h[0] == 'I' && h[1] == 'I') t.be = false;
    else if (h[0] == 'M' && h[1] == 'M') t.be = true;
    else return fail(t, "not a TIFF file (byte-order mark)");
    const uint64_t magic = r.uint(h + 2, 2);
    uint64_t ifd;
    if (magic == 42) {
        ifd = r.uint(h + 4, 4);
    } else if (magic == 43) {
        t.big = true;
        if (!r.get(0, h, 16) || r.uint(h + 4, 2) != 8) return fail(t, "bad BigTIFF header");
        ifd = r.uint(h + 8, 8);
    } else {
        return fail(t, "not a TIFF file (magic %llu)", (unsigned long long)magic);
    }
    const int cnt_sz = t.big ? 8 : 2, ent_sz = t.big ? 20 : 12, off_sz = t.big ? 8 : 4;
    int64_t nx = -1, ny = -1, nz = 0;
    int bits = 0, fmt = 1;
    uint64_t page_bytes = 0;
    std::vector<uint64_t> seen;
    while (ifd) {
        if (std::find(seen.begin(), seen.end(), ifd) != seen.end()) return fail(t, "IFD chain loops");
        if (seen.size() > (1u << 20)) return fail(t, "too many pages");
        seen.push_back(ifd);
        const uint64_t n = r.u(ifd, cnt_sz);
        if (!r.ok || n == 0 || n > 4096) return fail(t, "bad IFD at offset %llu", (unsigned long long)ifd);
        Entry E[8];  // width, length, bits, compression, offsets, spp, rows/strip, counts
        Entry pred, sfmt, planar, tilew;
        std::vector<unsigned char> ents(n * ent_sz);
        if (!r.get(ifd + cnt_sz, ents.data(), ents.size())) return fail(t, "truncated IFD");
        for (uint64_t i = 0; i < n; ++i) {
            const unsigned char *p = &ents[i * ent_sz];
            const int tag = (int)r.uint(p, 2);
            Entry e;
            e.type = (int)r.uint(p + 2, 2);
            e.count = r.uint(p + 4, off_sz);
            e.present = true;
            const int ts = type_size(e.type);
            const uint64_t val_pos = ifd + cnt_sz + i * ent_sz + 4 + off_sz;
            e.value_off = (ts && e.count * ts <= (uint64_t)off_sz) ? val_pos : r.uint(p + 4 + off_sz, off_sz);
            switch (tag) {
                case 256: E[0] = e; break;
                case 257: E[1] = e; break;
                case 258: E[2] = e; break;
                case 259: E[3] = e; break;
                case 273: E[4] = e; break;
                case 277: E[5] = e; break;
                case 278: E[6] = e; break;
                case 279: E[7] = e; break;
                case 284: planar = e; break;
                case 317: pred = e; break;
                case 322: tilew = e; break;
                case 339: sfmt = e; break;
                default: break;
            }
        }
        std::vector<uint64_t> v;
        auto one = [&](const Entry &e, uint64_t dflt) -> uint64_t {
            if (!e.present) return dflt;
            if (!tag_values(r, e, v) || v.empty()) return UINT64_MAX;
            return v[0];
        };
        const uint64_t w = one(E[0], 0), l = one(E[1], 0), b = one(E[2], 1), comp = one(E[3], 1),
                       spp = one(E[5], 1), pr = one(pred, 1), pl = one(planar, 1), sf = one(sfmt, 1);
        if (w == 0 || l == 0 || w == UINT64_MAX || l == UINT64_MAX) return fail(t, "page %zu: missing image size", seen.size() - 1);
        if (tilew.present) return fail(t, "tiled TIFF pages are not supported");
        if (comp != 1) return fail(t, "compression %llu is not supported (uncompressed only)", (unsigned long long)comp);
        if (pr != 1) return fail(t, "predictor %llu is not supported", (unsigned long long)pr);
        if (spp != 1 || (pl != 1 && pl != 2)) return fail(t, "%llu samples per pixel (grayscale only)", (unsigned long long)spp);
        if (!(b == 8 || b == 16 || b == 32 || b == 64)) return fail(t, "%llu bits per sample", (unsigned long long)b);
        if (!(sf == 1 || sf == 2 || sf == 3) || (sf == 3 && b < 32)) return fail(t, "sample format %llu / %llu bits", (unsigned long long)sf, (unsigned long long)b);
        if (nz == 0) {
            nx = (int64_t)w;
            ny = (int64_t)l;
            bits = (int)b;
            fmt = (int)sf;
            page_bytes = w * l * (b / 8);
        } else if ((int64_t)w != nx || (int64_t)l != ny || (int)b != bits || (int)sf != fmt) {
            return fail(t, "page %lld differs in size or sample type from page 0", (long long)nz);
        }
        std::vector<uint64_t> offs, cnts;
        if (!E[4].present || !tag_values(r, E[4], offs)) return fail(t, "page %lld: no strip offsets", (long long)nz);
        if (E[7].present) {
            if (!tag_values(r, E[7], cnts)) return fail(t, "page %lld: bad strip byte counts", (long long)nz);
        } else if (offs.size() == 1) {
            cnts.assign(1, page_bytes);
        } else {
            return fail(t, "page %lld: no strip byte counts", (long long)nz);
        }
        if (cnts.size() != offs.size()) return fail(t, "page %lld: strip tables differ in length", (long long)nz);
        const uint64_t rps = std::min<uint64_t>(one(E[6], l), l);
        const uint64_t row = w * (b / 8);
        uint64_t got = 0;
        for (size_t s = 0; s < offs.size() && got < page_bytes; ++s) {
            // a strip holds rps rows (the last one fewer); trailing pad bytes are ignored
            const uint64_t want = std::min<uint64_t>(rps == 0 ? page_bytes : rps * row, page_bytes - got);
            if (cnts[s] < want) return fail(t, "page %lld: strip %zu is short", (long long)nz, s);
            if (offs[s] + want > t.fsize) return fail(t, "page %lld: strip %zu past end of file", (long long)nz, s);
            t.segs.push_back({offs[s], want, (uint64_t)nz * page_bytes + got});
            got += want;
        }
        if (got != page_bytes) return fail(t, "page %lld: strips hold %llu of %llu bytes", (long long)nz, (unsigned long long)got, (unsigned long long)page_bytes);
        ++nz;
        ifd = r.u(ifd + cnt_sz + n * ent_sz, off_sz);
        if (!r.ok) return fail(t, "truncated IFD chain");
    }
    if (nz == 0) return fail(t, "no pages");
    // merge segments adjacent in the file and in the destination
    std::vector<Seg> m;
    for (const Seg &s : t.segs) {
        if (!m.empty() && m.back().file_off + m.back().len == s.file_off && m.back().dst_off + m.back().len == s.dst_off)
            m.back().len += s.len;
        else
            m.push_back(s);
    }
    t.segs.swap(m);
    t.info.nx = nx;
    t.info.ny = ny;
    t.info.nz = nz;
    t.info.bytes_per_sample = bits / 8;
    t.info.sample_format = fmt;
    t.info.big_endian = t.be ? 1 : 0;
    t.info.segments = (int64_t)t.segs.size();
    return CT_OK;
}

}  // namespace

extern "C" int ct_tiff_open(const char *path, ct_tiff_info *info, void **handle) {
    if (!path || !info || !handle) {
        ct::set_error("ct_tiff_open: null argument");
        return CT_ERR_PARAM;
    }
    *handle = nullptr;
    Tiff *t = new Tiff();
    t->path = path;
    t->fd = open(path, O_RDONLY | O_CLOEXEC);
    if (t->fd < 0) {
        const int st = fail(*t, "%s", strerror(errno));
        delete t;
        return st;
    }
    struct stat sb;
    if (fstat(t->fd, &sb) != 0) {
        const int st = fail(*t, "%s", strerror(errno));
        close(t->fd);
        delete t;
        return st;
    }
    t->fsize = (uint64_t)sb.st_size;
    const int st = parse(*t);
    if (st != CT_OK) {
        close(t->fd);
        delete t;
        return st;
    }
    *info = t->info;
    *handle = t;
    return CT_OK;
}

extern "C" int ct_tiff_read(void *handle, void *dst, int64_t dst_bytes, int32_t nthreads) {
    Tiff *t = (Tiff *)handle;
    if (!t || !dst) {
        ct::set_error("ct_tiff_read: null argument");
        return CT_ERR_PARAM;
    }
    const uint64_t need = (uint64_t)t->info.nx * t->info.ny * t->info.nz * t->info.bytes_per_sample;
    if ((uint64_t)dst_bytes < need) {
        ct::set_error("ct_tiff_read: destination holds %lld bytes, the stack needs %llu", (long long)dst_bytes,
                      (unsigned long long)need);
        return CT_ERR_PARAM;
    }
    // split the segments into ~equal byte ranges, one pread stream per thread
    constexpr uint64_t CHUNK = 8u << 20;
    std::vector<Seg> work;
    for (const Seg &s : t->segs)
        for (uint64_t o = 0; o < s.len; o += CHUNK)
            work.push_back({s.file_off + o, std::min(CHUNK, s.len - o), s.dst_off + o});
    const int nt = (int)std::max<int64_t>(1, std::min<int64_t>(std::max(nthreads, 1), (int64_t)work.size()));
    std::vector<int> err(nt, 0);
    auto run = [&](int id) {
        for (size_t i = id; i < work.size(); i += nt) {
            uint64_t done = 0;
            const Seg &s = work[i];
            while (done < s.len) {
                const ssize_t g = pread(t->fd, (char *)dst + s.dst_off + done, s.len - done, (off_t)(s.file_off + done));
                if (g <= 0) {
                    err[id] = g < 0 ? errno : EIO;
                    return;
                }
                done += (uint64_t)g;
            }
        }
    };
    if (nt == 1) {
        run(0);
    } else {
        std::vector<std::thread> th;
        for (int i = 0; i < nt; ++i) th.emplace_back(run, i);
        for (auto &x : th) x.join();
    }
    for (int e : err)
        if (e) return fail(*t, "read error: %s", strerror(e));
    return CT_OK;
}

extern "C" void ct_tiff_close(void *handle) {
    Tiff *t = (Tiff *)handle;
    if (!t) return;
    if (t->fd >= 0) close(t->fd);
    delete t;
}

namespace {

struct Out {
    std::vector<unsigned char> b;
    void put(uint64_t v, int n) {
        for (int i = 0; i < n; ++i) b.push_back((unsigned char)(v >> (8 * i)));
    }
};

}  // namespace

extern "C" int ct_tiff_write(const char *path, const void *src_zyx, int64_t nx, int64_t ny, int64_t nz,
                             int32_t bytes_per_sample, int32_t sample_format) {
    if (!path || !src_zyx || nx <= 0 || ny <= 0 || nz <= 0 || nx > UINT32_MAX || ny > UINT32_MAX ||
        !(bytes_per_sample == 1 || bytes_per_sample == 2 || bytes_per_sample == 4 || bytes_per_sample == 8) ||
        !(sample_format == 1 || sample_format == 2 || sample_format == 3)) {
        ct::set_error("ct_tiff_write: bad arguments");
        return CT_ERR_PARAM;
    }
    const uint64_t page = (uint64_t)nx * ny * bytes_per_sample, data = page * nz;
    char desc[128];
    snprintf(desc, sizeof desc, "{\"shape\": [%lld, %lld, %lld]}", (long long)nz, (long long)ny, (long long)nx);
    const uint64_t dlen = strlen(desc) + 1;
    const int NT = 11;  // entries per IFD
    const bool big = data + (uint64_t)nz * 256 + 4096 > 0xffffffffull;
    const int cnt_sz = big ? 8 : 2, ent_sz = big ? 20 : 12, off_sz = big ? 8 : 4;
    const uint64_t ifd_sz = cnt_sz + NT * ent_sz + off_sz;
    // layout: header | description | IFD 0..nz-1 | page data 0..nz-1 (contiguous)
    const uint64_t hdr = big ? 16 : 8, desc_off = hdr, ifd0 = (desc_off + dlen + 7) & ~7ull;
    const uint64_t data0 = (ifd0 + nz * ifd_sz + 15) & ~15ull;
    Out o;
    o.b.reserve(data0);
    o.put('I', 1);
    o.put('I', 1);
    if (big) {
        o.put(43, 2); o.put(8, 2); o.put(0, 2); o.put(ifd0, 8);
    } else {
        o.put(42, 2); o.put(ifd0, 4);
    }
    for (uint64_t i = 0; i < dlen; ++i) o.b.push_back(i + 1 < dlen ? (unsigned char)desc[i] : 0);
    o.b.resize(ifd0, 0);
    for (int64_t z = 0; z < nz; ++z) {
        const uint64_t at = ifd0 + z * ifd_sz;
        o.b.resize(at, 0);
        o.put(NT, cnt_sz);
        auto ent = [&](int tag, int type, uint64_t count, uint64_t value) {
            o.put(tag, 2);
            o.put(type, 2);
            o.put(count, off_sz);
            o.put(value, off_sz);
        };
        const int lt = big ? 16 : 4;  // LONG8 / LONG for offsets and counts
        ent(256, 4, 1, (uint64_t)nx);
        ent(257, 4, 1, (uint64_t)ny);
        ent(258, 3, 1, (uint64_t)bytes_per_sample * 8);
        ent(259, 3, 1, 1);
        ent(262, 3, 1, 1);  // minisblack
        ent(270, 2, z == 0 ? dlen : 1, z == 0 ? desc_off : 0);  // description on page 0 only
        ent(273, lt, 1, data0 + z * page);
        ent(277, 3, 1, 1);
        ent(278, 4, 1, (uint64_t)ny);
        ent(279, lt, 1, page);
        ent(339, 3, 1, (uint64_t)sample_format);
        o.put(z + 1 < nz ? at + ifd_sz : 0, off_sz);
    }
    o.b.resize(data0, 0);
    FILE *f = fopen(path, "wb");
    if (!f) {
        ct::set_error("failed to write image %s: %s", path, strerror(errno));
        return CT_ERR_IO;
    }
    bool ok = fwrite(o.b.data(), 1, o.b.size(), f) == o.b.size();
    ok = ok && fwrite(src_zyx, 1, data, f) == data;
    ok = (fclose(f) == 0) && ok;
    if (!ok) {
        ct::set_error("failed to write image %s: %s", path, strerror(errno));
        return CT_ERR_IO;
    }
    return CT_OK;
}
