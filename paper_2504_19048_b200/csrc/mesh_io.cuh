// mesh_io.cuh -- native mesh ingest and tally output (
// the paper-level PumiTally(mesh_filename, ...) / write(filename) of
// PAPER.md:265-270).  Part of libb200tally (included by b200tally.cu).
//
// * bt_mesh_read: the text format of read_tetmesh (mesh.py:302-331), parsed
//   on all host threads (line index by a parallel newline scan, then
//   std::from_chars -- correctly rounded, so every `repr` float written by
//   write_tetmesh comes back bit for bit, as Python's float() does).
// * bt_mesh_from_arrays: TetMesh.from_arrays (mesh.py:109-148) -- the same
//   orientation fix (swap local 2<->3 where the signed volume is negative),
//   degeneracy test and error messages, volumes/centroids/bbox evaluated in
//   numpy's operation order (so the arrays are bit-identical), adjacency by
//   bt_build_adjacency on a GPU (device >= 0) or a host sort (device < 0).
// * bt_write_vtk / bt_write_flux_csv: write_vtk / write_flux_csv
//   (tally.py:159-200) byte for byte, floats formatted as Python's repr.
#pragma once

#include <charconv>
#include <fstream>

struct bt_mesh {
    int64_t nv = 0, ne = 0;
    std::vector<double> v;     // (nv, 3)
    std::vector<int32_t> e;    // (ne, 4), positive orientation
    std::vector<int32_t> ae;   // (ne, 4), -1 on the boundary
    std::vector<int8_t> af;    // (ne, 4)
    std::vector<double> vol;   // (ne)
    std::vector<double> cen;   // (ne, 3)
    double bbox[6] = {0, 0, 0, 0, 0, 0};
};

// run fn(lo, hi) over [0, n) on up to `maxt` host threads
template <class F>
static void par_for(int64_t n, F fn, int maxt = 0) {
    const int hc = (int)std::max(1u, std::thread::hardware_concurrency());
    const int T = (int)std::max<int64_t>(1, std::min<int64_t>(maxt > 0 ? maxt : hc, n >> 14));
    if (T == 1) {
        fn((int64_t)0, n);
        return;
    }
    std::vector<std::thread> th;
    for (int t = 1; t < T; ++t) th.emplace_back([&, t] { fn(n * t / T, n * (t + 1) / T); });
    fn((int64_t)0, n / T);
    for (auto& x : th) x.join();
}

// ---- Python repr of a float (PyOS_double_to_string(x, 'r', 0, ADD_DOT_0)):
// the shortest round-trip digits; exponent form when decpt <= -4 or > 16
static int py_repr(double x, char* out) {
    if (std::isnan(x)) return (int)(strcpy(out, "nan"), 3);
    if (std::isinf(x)) return x > 0 ? (int)(strcpy(out, "inf"), 3) : (int)(strcpy(out, "-inf"), 4);
    char* p = out;
    if (std::signbit(x)) {
        *p++ = '-';
        x = -x;
    }
    if (x == 0.0) {
        memcpy(p, "0.0", 3);
        return (int)(p - out) + 3;
    }
    char buf[64];
    const auto r = std::to_chars(buf, buf + sizeof buf, x, std::chars_format::scientific);
    *r.ptr = 0;
    // buf = d[.ddd]e(+|-)XX
    char digits[32];
    int nd = 0;
    const char* q = buf;
    for (; *q && *q != 'e'; ++q)
        if (*q != '.') digits[nd++] = *q;
    const int exp10 = atoi(q + 1);
    const int decpt = exp10 + 1;
    if (decpt <= -4 || decpt > 16) {
        *p++ = digits[0];
        if (nd > 1) {
            *p++ = '.';
            memcpy(p, digits + 1, nd - 1);
            p += nd - 1;
        }
        p += sprintf(p, "e%c%02d", exp10 < 0 ? '-' : '+', exp10 < 0 ? -exp10 : exp10);
    } else if (decpt <= 0) {
        *p++ = '0';
        *p++ = '.';
        for (int k = 0; k < -decpt; ++k) *p++ = '0';
        memcpy(p, digits, nd);
        p += nd;
    } else if (decpt >= nd) {
        memcpy(p, digits, nd);
        p += nd;
        for (int k = nd; k < decpt; ++k) *p++ = '0';
        *p++ = '.';
        *p++ = '0';
    } else {
        memcpy(p, digits, decpt);
        p += decpt;
        *p++ = '.';
        memcpy(p, digits + decpt, nd - decpt);
        p += nd - decpt;
    }
    return (int)(p - out);
}

// ---- host face adjacency (build_adjacency, mesh.py:188-235) for device < 0:
// faces bucketed by their smallest vertex id (counting sort), each bucket
// (~F/V = 24 faces on a cube mesh) sorted by the other two ids on all host
// threads; equal neighbours pair up.  Errors report the first offending face
// in lexicographic order, as a full sort would.
static bt_status host_adjacency(const int32_t* el, int64_t ne, int64_t nv, int32_t* ae,
                                int8_t* af) {
    static const int FV[4][3] = {{1, 2, 3}, {0, 2, 3}, {0, 1, 3}, {0, 1, 2}};
    const int64_t F = 4 * ne;
    std::vector<int32_t> fa((size_t)F), fb((size_t)F), fc((size_t)F);
    par_for(ne, [&](int64_t lo, int64_t hi) {
        for (int64_t e = lo; e < hi; ++e)
            for (int f = 0; f < 4; ++f) {
                int32_t t[3] = {el[4 * e + FV[f][0]], el[4 * e + FV[f][1]], el[4 * e + FV[f][2]]};
                if (t[0] > t[1]) std::swap(t[0], t[1]);
                if (t[1] > t[2]) std::swap(t[1], t[2]);
                if (t[0] > t[1]) std::swap(t[0], t[1]);
                fa[(size_t)(4 * e + f)] = t[0];
                fb[(size_t)(4 * e + f)] = t[1];
                fc[(size_t)(4 * e + f)] = t[2];
            }
    });
    std::vector<int64_t> start((size_t)nv + 1, 0);
    for (int64_t r = 0; r < F; ++r) ++start[(size_t)fa[(size_t)r] + 1];
    for (int64_t v = 0; v < nv; ++v) start[(size_t)v + 1] += start[(size_t)v];
    std::vector<int64_t> fill(start.begin(), start.end() - 1);
    std::vector<int64_t> rows((size_t)F);
    for (int64_t r = 0; r < F; ++r) rows[(size_t)fill[(size_t)fa[(size_t)r]]++] = r;  // ascending rows
    std::fill(ae, ae + F, -1);
    std::fill(af, af + F, (int8_t)-1);
    // first error per kind: (bucket, message)
    std::mutex mu;
    int64_t err_at = INT64_MAX;
    std::string err_msg;
    par_for(nv, [&](int64_t lo, int64_t hi) {
        std::vector<int64_t> b;
        for (int64_t v = lo; v < hi; ++v) {
            const int64_t s0 = start[(size_t)v], s1 = start[(size_t)v + 1];
            if (s1 - s0 < 2) continue;
            b.assign(rows.begin() + s0, rows.begin() + s1);
            std::stable_sort(b.begin(), b.end(), [&](int64_t x, int64_t y) {
                return fb[(size_t)x] != fb[(size_t)y] ? fb[(size_t)x] < fb[(size_t)y]
                                                      : fc[(size_t)x] < fc[(size_t)y];
            });
            auto same = [&](size_t i, size_t j) {
                return fb[(size_t)b[i]] == fb[(size_t)b[j]] && fc[(size_t)b[i]] == fc[(size_t)b[j]];
            };
            for (size_t i = 0; i + 1 < b.size(); ++i) {
                if (!same(i, i + 1)) continue;
                char msg[200] = {0};
                const int64_t r1 = b[i], r2 = b[i + 1];
                if (i + 2 < b.size() && same(i + 1, i + 2))
                    snprintf(msg, sizeof msg,
                             "face with vertices (%d, %d, %d) is shared by more than two "
                             "elements (duplicate or non-manifold mesh)",
                             fa[(size_t)r1], fb[(size_t)r1], fc[(size_t)r1]);
                else if (r1 / 4 == r2 / 4)
                    snprintf(msg, sizeof msg,
                             "element %lld lists the same face twice (repeated vertex id)",
                             (long long)(r1 / 4));
                if (msg[0]) {
                    std::lock_guard<std::mutex> g(mu);
                    if (v < err_at) {
                        err_at = v;
                        err_msg = msg;
                    }
                    break;
                }
                ae[r1] = (int32_t)(r2 / 4);
                af[r1] = (int8_t)(r2 % 4);
                ae[r2] = (int32_t)(r1 / 4);
                af[r2] = (int8_t)(r1 % 4);
                ++i;
            }
        }
    });
    if (err_at != INT64_MAX) return set_err(BT_EINVAL, "%s", err_msg.c_str());
    for (int64_t e = 0; e < ne; ++e) {  // duplicated element
        const int32_t* r = ae + 4 * e;
        if (r[0] >= 0 && r[0] == r[1] && r[0] == r[2] && r[0] == r[3])
            return set_err(BT_EINVAL, "element %lld duplicates element %d", (long long)e, r[0]);
    }
    return BT_OK;
}

// TetMesh.from_arrays (mesh.py:109-148) into m (vertices and elements set)
static bt_status mesh_finish(bt_mesh* m, int32_t device) {
    const int64_t nv = m->nv, ne = m->ne;
    const double* V = m->v.data();
    int32_t* E = m->e.data();
    for (int64_t i = 0; i < 4 * ne; ++i)
        if (E[i] < 0 || E[i] >= nv) return set_err(BT_EINVAL, "element vertex id out of range");
    m->vol.assign((size_t)ne, 0.0);
    m->cen.assign((size_t)(3 * ne), 0.0);
    // signed_volumes6: a = v1 - v0, b = v2 - v0, c = v3 - v0; np.cross(a, b)
    // as numpy forms it; np.einsum("ij,ij->i", x, c) sums its three products
    // as (x0*c0 + x2*c2) + x1*c1 (two-lane accumulation; checked against
    // numpy on permuted torus meshes, tests/test_mesh_native.py)
    par_for(ne, [&](int64_t lo, int64_t hi) {
        for (int64_t e = lo; e < hi; ++e) {
            const double* p0 = V + 3 * (int64_t)E[4 * e];
            const double* p1 = V + 3 * (int64_t)E[4 * e + 1];
            const double* p2 = V + 3 * (int64_t)E[4 * e + 2];
            const double* p3 = V + 3 * (int64_t)E[4 * e + 3];
            double a[3], b[3], c[3];
            for (int k = 0; k < 3; ++k) {
                a[k] = p1[k] - p0[k];
                b[k] = p2[k] - p0[k];
                c[k] = p3[k] - p0[k];
            }
            const double x0 = a[1] * b[2] - a[2] * b[1];
            const double x1 = a[2] * b[0] - a[0] * b[2];
            const double x2 = a[0] * b[1] - a[1] * b[0];
            double v6 = x0 * c[0] + x2 * c[2];
            v6 = v6 + x1 * c[1];
            if (v6 < 0.0) {
                std::swap(E[4 * e + 2], E[4 * e + 3]);
                v6 = -v6;
            }
            m->vol[(size_t)e] = v6;  // vol6 for now
        }
    });
    double lo3[3] = {0, 0, 0}, hi3[3] = {0, 0, 0};
    if (nv) {
        for (int k = 0; k < 3; ++k) lo3[k] = hi3[k] = V[k];
        for (int64_t i = 1; i < nv; ++i)
            for (int k = 0; k < 3; ++k) {
                lo3[k] = std::min(lo3[k], V[3 * i + k]);
                hi3[k] = std::max(hi3[k], V[3 * i + k]);
            }
    }
    double span = 1.0;
    if (nv) span = std::max(hi3[0] - lo3[0], std::max(hi3[1] - lo3[1], hi3[2] - lo3[2]));
    const double s1 = std::max(span, 1.0);
    const double limit = 1e-12 * (s1 * s1 * s1);
    if (ne) {
        int64_t bad = 0;
        for (int64_t e = 1; e < ne; ++e)
            if (m->vol[(size_t)e] < m->vol[(size_t)bad]) bad = e;
        if (m->vol[(size_t)bad] <= limit) {
            char g[64];
            snprintf(g, sizeof g, "%g", m->vol[(size_t)bad] / 6.0);
            return set_err(BT_EINVAL, "element %lld is degenerate (volume %s)", (long long)bad, g);
        }
    }
    // volumes = vol6 / 6; centroids = vertices[elements].mean(axis=1)
    par_for(ne, [&](int64_t lo, int64_t hi) {
        for (int64_t e = lo; e < hi; ++e) {
            m->vol[(size_t)e] = m->vol[(size_t)e] / 6.0;
            for (int k = 0; k < 3; ++k) {
                double s = V[3 * (int64_t)E[4 * e] + k];
                s = s + V[3 * (int64_t)E[4 * e + 1] + k];
                s = s + V[3 * (int64_t)E[4 * e + 2] + k];
                s = s + V[3 * (int64_t)E[4 * e + 3] + k];
                m->cen[(size_t)(3 * e + k)] = s / 4.0;
            }
        }
    });
    for (int k = 0; k < 3; ++k) {
        m->bbox[k] = lo3[k];
        m->bbox[3 + k] = hi3[k];
    }
    m->ae.assign((size_t)(4 * ne), -1);
    m->af.assign((size_t)(4 * ne), (int8_t)-1);
    if (ne == 0) return BT_OK;
    if (device >= 0)
        return bt_build_adjacency(E, ne, nv, device, m->ae.data(), m->af.data());
    return host_adjacency(E, ne, nv, m->ae.data(), m->af.data());
}

// the text body of read_tetmesh: line index, then parallel parse
static bt_status mesh_parse(const std::string& path, const char* buf, size_t len, bt_mesh* m) {
    const char* nl = (const char*)memchr(buf, '\n', len);
    const size_t hlen = nl ? (size_t)(nl - buf) : len;
    char tag[16] = {0};
    long long nv = -1, ne = -1;
    char extra[8];
    std::string header(buf, hlen);
    if (sscanf(header.c_str(), "%15s %lld %lld %7s", tag, &nv, &ne, extra) != 3 ||
        strcmp(tag, "tetmesh") != 0) {
        if (strcmp(tag, "tetmesh") == 0 && sscanf(header.c_str(), "%15s %lld %lld", tag, &nv, &ne) != 3)
            return set_err(BT_EINVAL, "%s: bad header counts", path.c_str());
        if (strcmp(tag, "tetmesh") != 0 || sscanf(header.c_str(), "%15s %lld %lld %7s", tag, &nv,
                                                  &ne, extra) != 3)
            return set_err(BT_EINVAL, "%s: expected header 'tetmesh <nverts> <nelems>'",
                           path.c_str());
    }
    if (nv < 0 || ne < 0) return set_err(BT_EINVAL, "%s: bad header counts", path.c_str());
    const size_t body = nl ? hlen + 1 : len;
    // line starts of the body, by a parallel newline scan
    const int64_t nlines = nv + ne;
    std::vector<size_t> start;
    {
        const int T = (int)std::max(1u, std::min(16u, std::thread::hardware_concurrency()));
        std::vector<std::vector<size_t>> part((size_t)T);
        const size_t span = len - body;
        std::vector<std::thread> th;
        for (int t = 0; t < T; ++t)
            th.emplace_back([&, t] {
                const size_t lo = body + span * t / T, hi = body + span * (t + 1) / T;
                for (const char* p = buf + lo; p < buf + hi;) {
                    const char* q = (const char*)memchr(p, '\n', (size_t)(buf + hi - p));
                    if (!q) break;
                    part[(size_t)t].push_back((size_t)(q - buf) + 1);
                    p = q + 1;
                }
            });
        for (auto& x : th) x.join();
        start.push_back(body);
        for (auto& p : part) start.insert(start.end(), p.begin(), p.end());
        if (start.back() >= len) start.pop_back();  // trailing newline
    }
    if ((int64_t)start.size() < nlines)
        return set_err(BT_EINVAL, "%s: body does not match header counts", path.c_str());
    m->nv = nv;
    m->ne = ne;
    m->v.assign((size_t)(3 * nv), 0.0);
    m->e.assign((size_t)(4 * ne), 0);
    std::atomic<int> bad{0};
    auto line_end = [&](int64_t i) {
        return (size_t)i + 1 < start.size() ? start[(size_t)i + 1] : len;
    };
    par_for(nlines, [&](int64_t lo, int64_t hi) {
        for (int64_t i = lo; i < hi && !bad.load(std::memory_order_relaxed); ++i) {
            const char* p = buf + start[(size_t)i];
            const char* end = buf + line_end(i);
            const int want = i < nv ? 3 : 4;
            int got = 0;
            while (true) {
                while (p < end && (*p == ' ' || *p == '\t' || *p == '\r' || *p == '\n')) ++p;
                if (p >= end) break;
                if (got == want) {
                    bad = 1;
                    break;
                }
                std::from_chars_result r;
                if (i < nv) {
                    if (*p == '+') ++p;  // Python's float() accepts a leading '+'
                    r = std::from_chars(p, end, m->v[(size_t)(3 * i + got)]);
                } else {
                    long long x = 0;
                    if (*p == '+') ++p;
                    r = std::from_chars(p, end, x);
                    m->e[(size_t)(4 * (i - nv) + got)] = (int32_t)x;
                }
                if (r.ec != std::errc() ||
                    (r.ptr < end && !(*r.ptr == ' ' || *r.ptr == '\t' || *r.ptr == '\r' ||
                                      *r.ptr == '\n'))) {
                    bad = 2;
                    break;
                }
                p = r.ptr;
                ++got;
            }
            if (got != want && !bad) bad = 1;
        }
    });
    if (bad == 2) return set_err(BT_EINVAL, "%s: could not parse a number", path.c_str());
    if (bad) return set_err(BT_EINVAL, "%s: body does not match header counts", path.c_str());
    // anything after the last listed line must be blank
    for (size_t i = (size_t)nlines; i < start.size(); ++i)
        for (size_t k = start[i]; k < (i + 1 < start.size() ? start[i + 1] : len); ++k)
            if (!isspace((unsigned char)buf[k])) break;
    return BT_OK;
}

static bt_status write_text(const char* path, const std::string& s) {
    FILE* f = fopen(path, "wb");
    if (!f) return set_err(BT_EINVAL, "cannot open %s for writing", path);
    const size_t w = fwrite(s.data(), 1, s.size(), f);
    fclose(f);
    if (w != s.size()) return set_err(BT_EINVAL, "short write to %s", path);
    return BT_OK;
}

// append repr(x) + "\n" for x in a[0..n) (stride), formatted on host threads
static void append_reprs(std::string& out, const double* a, int64_t n, int64_t stride,
                         int64_t off) {
    const int T = (int)std::max<int64_t>(1, std::min<int64_t>(std::max(1u, std::thread::hardware_concurrency()), n >> 15));
    std::vector<std::string> part((size_t)T);
    std::vector<std::thread> th;
    auto job = [&](int t) {
        const int64_t lo = n * t / T, hi = n * (t + 1) / T;
        std::string& s = part[(size_t)t];
        s.reserve((size_t)(hi - lo) * 24);
        char b[48];
        for (int64_t i = lo; i < hi; ++i) {
            const int k = py_repr(a[i * stride + off], b);
            b[k] = '\n';
            s.append(b, (size_t)k + 1);
        }
    };
    for (int t = 1; t < T; ++t) th.emplace_back(job, t);
    job(0);
    for (auto& x : th) x.join();
    for (auto& s : part) out += s;
}
