// rr_bvh.cpp — binned-SAH BVH over a triangle soup (host, built once per
// scene upload; traversal is in rr_kernels.cu).
#include "rr_bvh.h"

#include <algorithm>
#include <cmath>
#include <cstring>

namespace rr {
namespace {

struct Box {
    float lo[3] = {INFINITY, INFINITY, INFINITY};
    float hi[3] = {-INFINITY, -INFINITY, -INFINITY};
    void grow(const float* p) {
        for (int k = 0; k < 3; ++k) {
            lo[k] = std::min(lo[k], p[k]);
            hi[k] = std::max(hi[k], p[k]);
        }
    }
    void grow(const Box& b) {
        for (int k = 0; k < 3; ++k) {
            lo[k] = std::min(lo[k], b.lo[k]);
            hi[k] = std::max(hi[k], b.hi[k]);
        }
    }
    float area() const {
        if (lo[0] > hi[0]) return 0.f;
        const float dx = hi[0] - lo[0], dy = hi[1] - lo[1], dz = hi[2] - lo[2];
        return 2.f * (dx * dy + dy * dz + dz * dx);
    }
};

struct Prim {
    Box box;
    float c[3];
    int index;
};

constexpr int kBins = 12;
constexpr int kLeafMax = 4;

float as_float(int v) {
    float f;
    std::memcpy(&f, &v, sizeof f);
    return f;
}

struct Builder {
    std::vector<Prim> prims;
    BvhBuild* out;
    const double* V;
    const int32_t* T;

    void emit_node(int idx, const Box& b, int a, int cnt) {
        float* n = &out->nodes[8 * (size_t)idx];
        n[0] = b.lo[0]; n[1] = b.lo[1]; n[2] = b.lo[2]; n[3] = as_float(a);
        n[4] = b.hi[0]; n[5] = b.hi[1]; n[6] = b.hi[2]; n[7] = as_float(cnt);
    }

    void emit_leaf(int idx, const Box& b, int first, int count) {
        const int tfirst = (int)(out->tris.size() / 12);
        for (int i = first; i < first + count; ++i) {
            const int t = prims[i].index;
            float v[3][3];
            for (int k = 0; k < 3; ++k)
                for (int c = 0; c < 3; ++c) v[k][c] = (float)V[3 * (size_t)T[3 * (size_t)t + k] + c];
            const float rec[12] = {v[0][0], v[0][1], v[0][2], as_float(t),
                                   v[1][0] - v[0][0], v[1][1] - v[0][1], v[1][2] - v[0][2], 0.f,
                                   v[2][0] - v[0][0], v[2][1] - v[0][1], v[2][2] - v[0][2], 0.f};
            out->tris.insert(out->tris.end(), rec, rec + 12);
        }
        emit_node(idx, b, tfirst, count);
    }

    void build(int idx, int first, int count, int depth) {
        out->depth = std::max(out->depth, depth);
        Box b, cb;
        for (int i = first; i < first + count; ++i) {
            b.grow(prims[i].box);
            cb.grow(prims[i].c);
        }
        if (count <= kLeafMax || depth >= 60) {
            emit_leaf(idx, b, first, count);
            return;
        }
        // binned SAH over centroids
        float best_cost = INFINITY;
        int best_axis = -1, best_split = -1;
        for (int ax = 0; ax < 3; ++ax) {
            const float ext = cb.hi[ax] - cb.lo[ax];
            if (!(ext > 0.f)) continue;
            Box bins[kBins];
            int cnt[kBins] = {0};
            for (int i = first; i < first + count; ++i) {
                int k = (int)((prims[i].c[ax] - cb.lo[ax]) / ext * kBins);
                k = std::min(std::max(k, 0), kBins - 1);
                bins[k].grow(prims[i].box);
                ++cnt[k];
            }
            float left_area[kBins];
            int left_cnt[kBins];
            Box acc;
            int n = 0;
            for (int k = 0; k < kBins; ++k) {
                acc.grow(bins[k]);
                n += cnt[k];
                left_area[k] = acc.area();
                left_cnt[k] = n;
            }
            acc = Box();
            n = 0;
            for (int k = kBins - 1; k > 0; --k) {
                acc.grow(bins[k]);
                n += cnt[k];
                const float cost = left_area[k - 1] * left_cnt[k - 1] + acc.area() * n;
                if (left_cnt[k - 1] > 0 && n > 0 && cost < best_cost) {
                    best_cost = cost;
                    best_axis = ax;
                    best_split = k;
                }
            }
        }
        int mid;
        if (best_axis < 0 || best_cost >= b.area() * count) {
            if (count <= 16 || best_axis < 0) {
                if (best_axis < 0) {   // all centroids coincide: median split
                    mid = first + count / 2;
                } else {
                    emit_leaf(idx, b, first, count);
                    return;
                }
            } else {
                mid = first + count / 2;
                const int ax = best_axis;
                std::nth_element(prims.begin() + first, prims.begin() + mid, prims.begin() + first + count,
                                 [ax](const Prim& x, const Prim& y) { return x.c[ax] < y.c[ax]; });
            }
        } else {
            const int ax = best_axis;
            const float ext = cb.hi[ax] - cb.lo[ax];
            auto it = std::partition(prims.begin() + first, prims.begin() + first + count,
                                     [&](const Prim& p) {
                                         int k = (int)((p.c[ax] - cb.lo[ax]) / ext * kBins);
                                         k = std::min(std::max(k, 0), kBins - 1);
                                         return k < best_split;
                                     });
            mid = (int)(it - prims.begin());
            if (mid == first || mid == first + count) mid = first + count / 2;
        }
        // children: left immediately follows, right after the left subtree
        const int left = (int)(out->nodes.size() / 8);
        out->nodes.resize(out->nodes.size() + 8);
        build(left, first, mid - first, depth + 1);
        const int right = (int)(out->nodes.size() / 8);
        out->nodes.resize(out->nodes.size() + 8);
        build(right, mid, first + count - mid, depth + 1);
        emit_node(idx, b, right, 0);
    }
};

} // namespace

void build_bvh(const double* vertices, int n_vertices, const int32_t* triangles, int n_triangles,
               BvhBuild& out) {
    (void)n_vertices;
    out = BvhBuild();
    Builder b;
    b.out = &out;
    b.V = vertices;
    b.T = triangles;
    b.prims.resize((size_t)n_triangles);
    for (int t = 0; t < n_triangles; ++t) {
        Prim& p = b.prims[(size_t)t];
        p.index = t;
        float c[3] = {0.f, 0.f, 0.f};
        for (int k = 0; k < 3; ++k) {
            float v[3];
            for (int a = 0; a < 3; ++a) v[a] = (float)vertices[3 * (size_t)triangles[3 * (size_t)t + k] + a];
            p.box.grow(v);
            for (int a = 0; a < 3; ++a) c[a] += v[a] / 3.f;
        }
        std::memcpy(p.c, c, sizeof c);
    }
    out.nodes.resize(8);
    out.tris.reserve((size_t)n_triangles * 12);
    if (n_triangles > 0) b.build(0, 0, n_triangles, 0);
}

} // namespace rr
