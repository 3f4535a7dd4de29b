// Scene ingestion: the reference's OBJ reader
// (scene.py:255-280 _parse_obj: positions only, fan triangulation, 1-based
// and negative indices, the current `g` / `o` / `usemtl` name per triangle)
// restated natively, so a million-triangle mesh loads in a fraction of a
// second instead of a per-line Python loop.  Numbers are parsed with strtod /
// strtoll (correctly rounded, like Python's float() / int(), including the
// digit-separating underscores Python accepts).  The parsed arrays are then
// the soup load_scene hands to ef_scene_create_ex (host SAH or device LBVH).
#include <cerrno>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <unordered_map>
#include <vector>

#include "ef_internal.h"

struct ef_mesh {
    std::vector<double> verts;        // (V, 3)
    std::vector<int64_t> tris;        // (T, 3) 0-based
    std::vector<int32_t> tri_group;   // (T) index into names
    std::vector<std::string> names;   // group names ("" = none)
};

namespace {

bool is_space(char c) { return c == ' ' || c == '\t' || c == '\r' || c == '\n' || c == '\f' || c == '\v'; }

// Python-style underscores: allowed only between two digits.
bool strip_underscores(const std::string& in, std::string& out) {
    out.clear();
    for (size_t i = 0; i < in.size(); ++i) {
        if (in[i] == '_') {
            if (i == 0 || i + 1 >= in.size() || !isdigit((unsigned char)in[i - 1]) ||
                !isdigit((unsigned char)in[i + 1]))
                return false;
            continue;
        }
        out.push_back(in[i]);
    }
    return true;
}

// Token [b, e) of a NUL-terminated buffer (whitespace after e).  Fast path:
// strtod / strtoll straight on the buffer; tokens with '_' go through the
// Python underscore rule first.
bool parse_double(const char* b, const char* e, double& v) {
    // Python's float() takes no hexadecimal literals (strtod would)
    if (std::memchr(b, 'x', e - b) || std::memchr(b, 'X', e - b)) return false;
    if (std::memchr(b, '_', e - b)) {
        std::string s;
        if (!strip_underscores(std::string(b, e), s) || s.empty()) return false;
        char* end = nullptr;
        v = std::strtod(s.c_str(), &end);
        return end == s.c_str() + s.size();
    }
    char* end = nullptr;
    v = std::strtod(b, &end);   // overflow -> +-inf like Python's float('1e999')
    return end == e && e > b;
}

bool parse_int(const char* b, const char* e, long long& v) {
    if (std::memchr(b, '_', e - b)) {
        std::string s;
        if (!strip_underscores(std::string(b, e), s) || s.empty()) return false;
        char* end = nullptr;
        errno = 0;
        v = std::strtoll(s.c_str(), &end, 10);
        return end == s.c_str() + s.size() && errno == 0;
    }
    char* end = nullptr;
    errno = 0;
    v = std::strtoll(b, &end, 10);
    return end == e && e > b && errno == 0;
}

}  // namespace

using ef::set_error;

extern "C" int ef_obj_parse(const char* path, ef_mesh** out) {
    if (!path || !out) return set_error(EF_EINVAL, "ef_obj_parse: null argument");
    *out = nullptr;
    FILE* f = std::fopen(path, "rb");
    if (!f) return set_error(EF_EINVAL, std::string("ef_obj_parse: cannot open ") + path);
    std::vector<char> text;
    {   // the whole file, NUL-terminated (tokens are parsed in place)
        char buf[1 << 20];
        size_t n;
        while ((n = std::fread(buf, 1, sizeof buf, f)) > 0) text.insert(text.end(), buf, buf + n);
        std::fclose(f);
        text.push_back('\n');
        text.push_back('\0');
    }
    ef_mesh* m = new ef_mesh();
    std::unordered_map<std::string, int32_t> group_id;
    auto gid = [&](const std::string& name) {
        auto it = group_id.find(name);
        if (it != group_id.end()) return it->second;
        const int32_t id = (int32_t)m->names.size();
        m->names.push_back(name);
        group_id.emplace(name, id);
        return id;
    };
    int32_t current = gid("");
    std::vector<const char*> tb, te;   // token bounds of the current line
    std::vector<long long> idx;
    long long lineno = 0;
    std::string err;
    const char* p = text.data();
    const char* const end = text.data() + text.size() - 1;   // at the final NUL
    while (p < end && err.empty()) {
        const char* eol = static_cast<const char*>(std::memchr(p, '\n', end - p));
        if (!eol) eol = end;
        ++lineno;
        tb.clear();
        te.clear();
        for (const char* q = p; q < eol;) {   // str.split()
            while (q < eol && is_space(*q)) ++q;
            const char* j = q;
            while (q < eol && !is_space(*q)) ++q;
            if (q > j) {
                tb.push_back(j);
                te.push_back(q);
            }
        }
        p = eol + 1;
        if (tb.empty() || tb[0][0] == '#') continue;
        const size_t taglen = te[0] - tb[0];
        auto tag_is = [&](const char* t) { return taglen == std::strlen(t) && !std::memcmp(tb[0], t, taglen); };
        if (tag_is("v")) {
            if (tb.size() < 4) {
                err = "vertex with fewer than 3 coordinates";
                break;
            }
            for (int k = 1; k <= 3; ++k) {
                double v;
                if (!parse_double(tb[k], te[k], v)) {
                    err = "bad vertex coordinate '" + std::string(tb[k], te[k]) + "'";
                    break;
                }
                m->verts.push_back(v);
            }
        } else if (tag_is("g") || tag_is("o") || tag_is("usemtl")) {
            current = gid(tb.size() > 1 ? std::string(tb[1], te[1]) : std::string());
        } else if (tag_is("f")) {
            idx.clear();
            const long long nv = (long long)(m->verts.size() / 3);
            for (size_t k = 1; k < tb.size(); ++k) {
                const char* slash = static_cast<const char*>(std::memchr(tb[k], '/', te[k] - tb[k]));
                long long i;
                if (!parse_int(tb[k], slash ? slash : te[k], i)) {
                    err = "bad face index '" + std::string(tb[k], te[k]) + "'";
                    break;
                }
                i = i > 0 ? i - 1 : nv + i;
                if (i < 0 || i >= nv) {   // the reference fails later with an IndexError
                    err = "face index '" + std::string(tb[k], te[k]) + "' out of range";
                    break;
                }
                idx.push_back(i);
            }
            if (!err.empty()) break;
            for (size_t k = 1; k + 1 < idx.size(); ++k) {   // fan triangulation
                m->tris.push_back(idx[0]);
                m->tris.push_back(idx[k]);
                m->tris.push_back(idx[k + 1]);
                m->tri_group.push_back(current);
            }
        }
    }
    if (!err.empty()) {
        delete m;
        return set_error(EF_EINVAL, "ef_obj_parse: " + std::string(path) + ":" + std::to_string(lineno) +
                                        ": " + err);
    }
    *out = m;
    return EF_OK;
}

extern "C" int ef_mesh_info(const ef_mesh* m, int64_t* out4) {
    if (!m || !out4) return set_error(EF_EINVAL, "ef_mesh_info: null argument");
    out4[0] = (int64_t)(m->verts.size() / 3);
    out4[1] = (int64_t)m->tri_group.size();
    out4[2] = (int64_t)m->names.size();
    int64_t bytes = 0;
    for (const auto& n : m->names) bytes += (int64_t)n.size() + 1;
    out4[3] = bytes;
    return EF_OK;
}

extern "C" int ef_mesh_arrays(const ef_mesh* m, double* verts, int64_t* tris, int32_t* tri_group,
                              char* names, int64_t names_bytes) {
    if (!m) return set_error(EF_EINVAL, "ef_mesh_arrays: null mesh");
    if (verts && !m->verts.empty()) std::memcpy(verts, m->verts.data(), m->verts.size() * sizeof(double));
    if (tris && !m->tris.empty()) std::memcpy(tris, m->tris.data(), m->tris.size() * sizeof(int64_t));
    if (tri_group && !m->tri_group.empty())
        std::memcpy(tri_group, m->tri_group.data(), m->tri_group.size() * sizeof(int32_t));
    if (names) {
        int64_t o = 0;
        for (const auto& n : m->names) {
            if (o + (int64_t)n.size() + 1 > names_bytes)
                return set_error(EF_EINVAL, "ef_mesh_arrays: names buffer too small");
            std::memcpy(names + o, n.c_str(), n.size() + 1);
            o += (int64_t)n.size() + 1;
        }
    }
    return EF_OK;
}

extern "C" int ef_mesh_destroy(ef_mesh* m) {
    delete m;
    return EF_OK;
}
