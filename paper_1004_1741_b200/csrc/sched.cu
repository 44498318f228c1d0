// sched.cu -- work schedules of the temporally blocked Jacobi launch (host
// only).  A launch processes (tile, k-range) items; persistent CTAs claim
// them in order from an atomic counter (jacobi_tb.cuh: decode_item).  This
// file decides the items: either the regular k-block-major decomposition
// (one block length for the launch, decoded arithmetically) or an explicit
// list uploaded once per launch shape.
//
// Cost model (fitted on B200 at 1024^3, T=4: k-block lengths 128..1024
// predict the measured launch times to +-1.5%): an item of `len` output
// planes costs len + 2T (trapezoid warm-up) + 4 (item switch) plane steps;
// the makespan is that of the greedy claim order (first free CTA takes the
// next item).
#include <cuda_runtime.h>

#include <algorithm>
#include <climits>
#include <cstdint>
#include <cstdlib>
#include <map>
#include <mutex>
#include <queue>
#include <tuple>
#include <vector>

#include "../../include/stencil_b200.h"
#include "sb_internal.h"

namespace sb {

namespace {

struct Item {
    int tile, k0, k1;
    double cost;
};

double env_double(const char* name, double dflt) {
    const char* v = tune_env(name);
    return v ? atof(v) : dflt;
}

int env_int(const char* name, int dflt) {
    const char* v = tune_env(name);
    return v ? atoi(v) : dflt;
}

double span_of(const std::vector<Item>& items, int grid) {
    std::priority_queue<double, std::vector<double>, std::greater<double>> q;
    for (int c = 0; c < grid; ++c) q.push(0.0);
    double span = 0;
    for (const Item& it : items) {
        const double f = q.top() + it.cost;
        q.pop();
        q.push(f);
        span = std::max(span, f);
    }
    return span;
}

}  // namespace

// Work-item length along k for the regular decomposition.
//  * T = 1, 2 (HBM-bound): short blocks.  Work items are handed out
//    k-block-major, so short blocks keep every resident CTA within a few
//    planes of each other and the overlapping halo rows/columns that
//    neighbouring tiles re-read hit L2 (measured on B200, 1024^3: T=1 327 ->
//    382 GLUP/s at 8 planes; T=2 605 -> 618 at 64).
//  * T >= 3 (compute-bound): among the block lengths ceil(nk / nb) and the
//    "about 8 items per CTA" length, the one minimising the modelled
//    makespan.
int64_t schedule_span(int T, int tiles, int nkout, int grid, int kb) {
    std::priority_queue<int64_t, std::vector<int64_t>, std::greater<int64_t>> q;
    for (int c = 0; c < grid; ++c) q.push(0);
    int64_t span = 0;
    for (int blk = 0; (int64_t)blk * kb < nkout; ++blk) {
        const int64_t cost = std::min(kb, nkout - blk * kb) + 2 * T + 4;
        for (int t = 0; t < tiles; ++t) {
            const int64_t f = q.top() + cost;
            q.pop();
            q.push(f);
            span = std::max(span, f);
        }
    }
    return span;
}

int pick_kblock(int T, int tiles, int nkout, int grid) {
    if (T == 1) return 8;
    if (T == 2) return 64;
    static std::mutex mu;
    static std::map<std::tuple<int, int, int, int>, int> cache;
    const auto key = std::make_tuple(T, tiles, nkout, grid);
    {
        std::lock_guard<std::mutex> lk(mu);
        auto it = cache.find(key);
        if (it != cache.end()) return it->second;
    }
    const int64_t want = (int64_t)grid * 8;
    int kb0 = (int)std::min<int64_t>(((int64_t)tiles * nkout + want - 1) / want, nkout);
    kb0 = std::max(kb0, std::min(8 * T, nkout));
    std::vector<int> cands{kb0};
    for (int nb = 1; nb <= 64; ++nb) {
        const int kb = (nkout + nb - 1) / nb;
        if (kb < 4 * T && nb > 1) break;
        cands.push_back(kb);
    }
    int best_kb = kb0;
    int64_t best = INT64_MAX;
    for (int kb : cands) {
        const int64_t sp = schedule_span(T, tiles, nkout, grid, kb);
        if (sp < best || (sp == best && kb > best_kb)) {
            best = sp;
            best_kb = kb;
        }
    }
    std::lock_guard<std::mutex> lk(mu);
    cache[key] = best_kb;
    return best_kb;
}

// Explicit schedules for T >= 3 (SB_LIST selects; default 1):
//   1: whole-k "bulk" rounds (border tiles first), tail = the leftover tiles
//      cut into m * grid k-pieces (m = SB_LIST_M or the model's best)
//   2: (rounds - 1) bulk rounds, then the remaining tiles k-block-major with
//      the block length the model picks (SB_LIST_KB overrides)
// Border tiles (MASK step mode) cost SB_SELF (default 1.2) x a FAST tile.
static std::vector<Item> build_list(int mode, int T, int tiles_i, int tiles_j,
                                    const std::vector<char>& border, int kfirst, int klast,
                                    int grid, int m_or_kb) {
    const int tiles = tiles_i * tiles_j, nk = klast - kfirst;
    const double f = env_double("SB_SELF", 1.2);
    auto cost = [&](int t, int len) { return (len + 2.0 * T + 4.0) * (border[t] ? f : 1.0); };
    // tile order: border tiles first (longest first), then the rest
    std::vector<int> order;
    for (int t = 0; t < tiles; ++t)
        if (border[t]) order.push_back(t);
    for (int t = 0; t < tiles; ++t)
        if (!border[t]) order.push_back(t);
    std::vector<Item> items;
    int rounds = tiles / grid;
    if (mode == 2 && rounds > 0) --rounds;
    const int nbulk = rounds * grid;
    for (int x = 0; x < nbulk; ++x) items.push_back({order[x], kfirst, klast, cost(order[x], nk)});
    const int R = tiles - nbulk;
    if (R == 0) return items;
    if (mode == 1) {
        const int P = m_or_kb * grid;
        if (P < R) return {};
        for (int r = 0; r < R; ++r) {
            const int t = order[nbulk + r];
            const int pieces = std::min(nk, P / R + (r < P % R ? 1 : 0));
            for (int q = 0; q < pieces; ++q) {
                const int k0 = kfirst + (int)((int64_t)nk * q / pieces);
                const int k1 = kfirst + (int)((int64_t)nk * (q + 1) / pieces);
                items.push_back({t, k0, k1, cost(t, k1 - k0)});
            }
        }
    } else {
        const int kb = std::max(1, std::min(m_or_kb, nk));
        for (int k0 = kfirst; k0 < klast; k0 += kb) {
            const int k1 = std::min(k0 + kb, klast);
            for (int r = 0; r < R; ++r) {
                const int t = order[nbulk + r];
                items.push_back({t, k0, k1, cost(t, k1 - k0)});
            }
        }
    }
    return items;
}

// The explicit list for this launch shape, or empty when the regular
// k-block decomposition (block length kb) is at least as good under the
// model.  Host only; deterministic.
std::vector<int4> build_item_list(int T, int tiles_i, int tiles_j, const std::vector<char>& border,
                                  int kfirst, int klast, int grid, int kb) {
    const int mode = env_int("SB_LIST", 1);
    if (T < 3 || mode == 0 || klast <= kfirst) return {};
    const int tiles = tiles_i * tiles_j, nk = klast - kfirst;
    const double f = env_double("SB_SELF", 1.2);
    // the regular schedule under the same (border-aware) model
    std::vector<Item> reg;
    for (int k0 = kfirst; k0 < klast; k0 += kb)
        for (int t = 0; t < tiles; ++t) {
            const int k1 = std::min(k0 + kb, klast);
            reg.push_back({t, k0, k1, (k1 - k0 + 2.0 * T + 4.0) * (border[t] ? f : 1.0)});
        }
    double best_span = span_of(reg, grid);
    std::vector<Item> best;
    std::vector<int> params;
    if (mode == 1) {
        const int m = env_int("SB_LIST_M", 0);
        if (m > 0) params.push_back(m);
        else params = {1, 2, 3, 4, 6, 8};
    } else {
        const int k = env_int("SB_LIST_KB", 0);
        if (k > 0) params.push_back(k);
        else
            for (int nb = 1; nb <= 32; ++nb) params.push_back((nk + nb - 1) / nb);
    }
    const bool force = tune_env("SB_LIST_FORCE") != nullptr;
    for (int prm : params) {
        std::vector<Item> v = build_list(mode, T, tiles_i, tiles_j, border, kfirst, klast, grid, prm);
        if (v.empty()) continue;
        const double sp = span_of(v, grid);
        if (sp < best_span || (force && best.empty())) {
            best_span = sp;
            best.swap(v);
        }
    }
    std::vector<int4> h;
    for (const Item& x : best) h.push_back(make_int4(x.tile, x.k0, x.k1, 0));
    return h;
}

int item_list(int T, int tiles_i, int tiles_j, const std::vector<char>& border, int kfirst,
              int klast, int grid, int kb, bool regular_only, const int4** out, int* count) {
    *out = nullptr;
    *count = 0;
    const int mode = env_int("SB_LIST", 1);
    if (T < 3) return SB_OK;  // T = 1, 2: short regular k-blocks, decoded arithmetically
    int dev;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return cuda_fail(e, "cudaGetDevice");
    static std::mutex mu;
    static std::map<std::tuple<int, int, int, int, int, int, int, int, int, std::vector<char>>,
                    std::pair<int4*, int>>
        cache;
    const auto key = std::make_tuple(dev, T, tiles_i, tiles_j, kfirst, klast, grid,
                                     regular_only ? -1 : mode, kb, border);
    std::lock_guard<std::mutex> lk(mu);
    auto it = cache.find(key);
    if (it == cache.end()) {
        std::vector<int4> h;
        if (!regular_only) h = build_item_list(T, tiles_i, tiles_j, border, kfirst, klast, grid, kb);
        // where the model prefers the regular decomposition it is uploaded as
        // a list too, in claim order (k-block major): kernels of depth >= 3
        // decode items from a list only
        if (h.empty())
            for (int k0 = kfirst; k0 < klast; k0 += std::max(kb, 1))
                for (int t = 0; t < tiles_i * tiles_j; ++t)
                    h.push_back(make_int4(t, k0, std::min(k0 + std::max(kb, 1), klast), 0));
        int4* d = nullptr;
        if (!h.empty()) {
            e = cudaMalloc(&d, h.size() * sizeof(int4));
            if (e != cudaSuccess) return cuda_fail(e, "cudaMalloc(item list)");
            e = cudaMemcpy(d, h.data(), h.size() * sizeof(int4), cudaMemcpyHostToDevice);
            if (e != cudaSuccess) return cuda_fail(e, "cudaMemcpy(item list)");
        }
        it = cache.emplace(key, std::make_pair(d, (int)h.size())).first;
    }
    *out = it->second.first;
    *count = it->second.second;
    return SB_OK;
}

}  // namespace sb
