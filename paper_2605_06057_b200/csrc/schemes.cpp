// schemes.cpp -- built-in LCMA coefficient tables, composition, Brent
// validation and the text loader of the product library.  Written
// independently of oracle/ (different encoding, different code); the tests
// check the two against each other and against the Brent identity.
#include "schemes.h"

#include <algorithm>
#include <cstdlib>
#include <memory>
#include <mutex>
#include <sstream>

#include "../../include/lcma.h"

namespace lcma {

int Scheme::nnzU() const { int c = 0; for (auto x : U) c += (x != 0); return c; }
int Scheme::nnzV() const { int c = 0; for (auto x : V) c += (x != 0); return c; }
int Scheme::nnzW() const { int c = 0; for (auto x : W) c += (x != 0); return c; }

namespace {

Scheme make_classical() {
    Scheme s;
    s.name = "classical";
    s.m = s.k = s.n = s.R = 1;
    s.U = {1};
    s.V = {1};
    s.W = {1};
    return s;
}

// Strassen 1969, classic numbering: rows are products r=1..7,
// columns the 2x2 blocks in row-major order (11, 12, 21, 22).
Scheme make_strassen() {
    static const int8_t U[7][4] = {{1, 0, 0, 1}, {0, 0, 1, 1}, {1, 0, 0, 0}, {0, 0, 0, 1},
                                   {1, 1, 0, 0}, {-1, 0, 1, 0}, {0, 1, 0, -1}};
    static const int8_t V[7][4] = {{1, 0, 0, 1}, {1, 0, 0, 0}, {0, 1, 0, -1}, {-1, 0, 1, 0},
                                   {0, 0, 0, 1}, {1, 1, 0, 0}, {0, 0, 1, 1}};
    static const int8_t W[7][4] = {{1, 0, 0, 1}, {0, 0, 1, -1}, {0, 1, 0, 1}, {1, 0, 1, 0},
                                   {-1, 1, 0, 0}, {0, 0, 0, 1}, {1, 0, 0, 0}};
    Scheme s;
    s.name = "strassen-2x2x2-r7";
    s.m = s.k = s.n = 2;
    s.R = 7;
    for (int r = 0; r < 7; ++r)
        for (int b = 0; b < 4; ++b) {
            s.U.push_back(U[r][b]);
            s.V.push_back(V[r][b]);
            s.W.push_back(W[r][b]);
        }
    return s;
}

// Laderman 1976 <3,3,3;23>.  Each factor is a 0-terminated list of
// signed two-digit block codes (row*10 + col, 1-based).
Scheme make_laderman() {
    static const int Ua[23][8] = {
        {11, 12, 13, -21, -22, -32, -33, 0}, {11, -21, 0}, {22, 0}, {-11, 21, 22, 0},
        {21, 22, 0}, {11, 0}, {-11, 31, 32, 0}, {-11, 31, 0}, {31, 32, 0},
        {11, 12, 13, -22, -23, -31, -32, 0}, {32, 0}, {-13, 32, 33, 0}, {13, -33, 0},
        {13, 0}, {32, 33, 0}, {-13, 22, 23, 0}, {13, -23, 0}, {22, 23, 0}, {12, 0},
        {23, 0}, {21, 0}, {31, 0}, {33, 0}};
    static const int Vb[23][8] = {
        {22, 0}, {-12, 22, 0}, {-11, 12, 21, -22, -23, -31, 33, 0}, {11, -12, 22, 0},
        {-11, 12, 0}, {11, 0}, {11, -13, 23, 0}, {13, -23, 0}, {-11, 13, 0}, {23, 0},
        {-11, 13, 21, -22, -23, -31, 32, 0}, {22, 31, -32, 0}, {22, -32, 0}, {31, 0},
        {-31, 32, 0}, {23, 31, -33, 0}, {23, -33, 0}, {-31, 33, 0}, {21, 0}, {32, 0},
        {13, 0}, {12, 0}, {33, 0}};
    // C_ij = sum of the listed products (all +1), 0-terminated.
    static const int Cm[9][8] = {
        {6, 14, 19, 0},            {1, 4, 5, 6, 12, 14, 15},  {6, 7, 9, 10, 14, 16, 18},
        {2, 3, 4, 6, 14, 16, 17},  {2, 4, 5, 6, 20, 0},       {14, 16, 17, 18, 21, 0},
        {6, 7, 8, 11, 12, 13, 14}, {12, 13, 14, 15, 22, 0},   {6, 7, 8, 9, 23, 0}};
    Scheme s;
    s.name = "laderman-3x3x3-r23";
    s.m = s.k = s.n = 3;
    s.R = 23;
    s.U.assign(23 * 9, 0);
    s.V.assign(23 * 9, 0);
    s.W.assign(23 * 9, 0);
    auto put = [](std::vector<int8_t>& T, int r, const int* codes) {
        for (int t = 0; t < 8 && codes[t]; ++t) {
            int c = codes[t], sg = c < 0 ? -1 : 1;
            c = std::abs(c);
            int i = c / 10 - 1, j = c % 10 - 1;
            T[r * 9 + i * 3 + j] = (int8_t)sg;
        }
    };
    for (int r = 0; r < 23; ++r) {
        put(s.U, r, Ua[r]);
        put(s.V, r, Vb[r]);
    }
    for (int ij = 0; ij < 9; ++ij)
        for (int t = 0; t < 7 && Cm[ij][t]; ++t) s.W[(Cm[ij][t] - 1) * 9 + ij] = 1;
    return s;
}

struct Registry {
    std::mutex mu;
    std::vector<Scheme> all;
    Registry() {
        all.reserve(256);   // pointers from scheme_get() must stay valid
        all.push_back(make_classical());
        Scheme st = make_strassen();
        all.push_back(st);
        Scheme s2 = scheme_compose(st, st);
        s2.name = "strassen2-4x4x4-r49";
        all.push_back(s2);
        all.push_back(make_laderman());
        for (int i = 0; i < (int)all.size(); ++i) all[i].id = i;
        all[2].base_id = 1;   // Strassen^2 = Strassen o Strassen
    }
};

Registry& reg() {
    static Registry r;
    return r;
}

}  // namespace

Scheme scheme_compose(const Scheme& a, const Scheme& b) {
    // Two-level scheme: r = r1*R2 + r2, block index i = i1*m2 + i2
    // (outer-major), coefficients multiply ("two-level recursive").
    Scheme s;
    s.name = a.name + "*" + b.name;
    s.m = a.m * b.m;
    s.k = a.k * b.k;
    s.n = a.n * b.n;
    s.R = a.R * b.R;
    s.U.assign((size_t)s.R * s.m * s.k, 0);
    s.V.assign((size_t)s.R * s.k * s.n, 0);
    s.W.assign((size_t)s.R * s.m * s.n, 0);
    for (int r1 = 0; r1 < a.R; ++r1)
        for (int r2 = 0; r2 < b.R; ++r2) {
            const int r = r1 * b.R + r2;
            for (int i1 = 0; i1 < a.m; ++i1)
                for (int i2 = 0; i2 < b.m; ++i2)
                    for (int l1 = 0; l1 < a.k; ++l1)
                        for (int l2 = 0; l2 < b.k; ++l2)
                            s.U[((size_t)r * s.m + i1 * b.m + i2) * s.k + l1 * b.k + l2] =
                                (int8_t)(a.u(r1, i1, l1) * b.u(r2, i2, l2));
            for (int l1 = 0; l1 < a.k; ++l1)
                for (int l2 = 0; l2 < b.k; ++l2)
                    for (int j1 = 0; j1 < a.n; ++j1)
                        for (int j2 = 0; j2 < b.n; ++j2)
                            s.V[((size_t)r * s.k + l1 * b.k + l2) * s.n + j1 * b.n + j2] =
                                (int8_t)(a.v(r1, l1, j1) * b.v(r2, l2, j2));
            for (int i1 = 0; i1 < a.m; ++i1)
                for (int i2 = 0; i2 < b.m; ++i2)
                    for (int j1 = 0; j1 < a.n; ++j1)
                        for (int j2 = 0; j2 < b.n; ++j2)
                            s.W[((size_t)r * s.m + i1 * b.m + i2) * s.n + j1 * b.n + j2] =
                                (int8_t)(a.w(r1, i1, j1) * b.w(r2, i2, j2));
        }
    return s;
}

long long scheme_brent_failures(const Scheme& s, std::string* first) {
    // sum_r U[r,i,l] V[r,l',j] W[r,i',j'] must equal [i=i'][l=l'][j=j'].
    long long fails = 0;
    for (int i = 0; i < s.m; ++i)
        for (int l = 0; l < s.k; ++l)
            for (int l2 = 0; l2 < s.k; ++l2)
                for (int j = 0; j < s.n; ++j)
                    for (int i2 = 0; i2 < s.m; ++i2)
                        for (int j2 = 0; j2 < s.n; ++j2) {
                            long long acc = 0;
                            for (int r = 0; r < s.R; ++r)
                                acc += (long long)s.u(r, i, l) * s.v(r, l2, j) * s.w(r, i2, j2);
                            long long want = (i == i2 && l == l2 && j == j2) ? 1 : 0;
                            if (acc != want) {
                                if (fails == 0 && first) {
                                    std::ostringstream os;
                                    os << "Brent identity fails at (i,l,l',j,i',j')=(" << i << ","
                                       << l << "," << l2 << "," << j << "," << i2 << "," << j2
                                       << "): sum=" << acc << " expected " << want;
                                    *first = os.str();
                                }
                                ++fails;
                            }
                        }
    return fails;
}

const Scheme* scheme_get(int id) {
    Registry& R = reg();
    std::lock_guard<std::mutex> g(R.mu);
    if (id < 0 || id >= (int)R.all.size()) return nullptr;
    return &R.all[id];   // elements are never removed; deque-like stability below
}

int scheme_register(const Scheme& s, std::string& err) {
    if (s.m < 1 || s.k < 1 || s.n < 1 || s.R < 1) {
        err = "scheme dimensions must be >= 1";
        return -LCMA_ERR_INVALID_VALUE;
    }
    if (s.R > 128 || s.m * s.n > 32 || s.m * s.k > 32 || s.k * s.n > 32) {
        err = "scheme too large for this build (R <= 128, m*n, m*k, k*n <= 32)";
        return -LCMA_ERR_NOT_SUPPORTED;
    }
    if ((int)s.U.size() != s.R * s.m * s.k || (int)s.V.size() != s.R * s.k * s.n ||
        (int)s.W.size() != s.R * s.m * s.n) {
        err = "coefficient tensor shape mismatch";
        return -LCMA_ERR_INVALID_VALUE;
    }
    for (const auto* T : {&s.U, &s.V, &s.W})
        for (int8_t c : *T)
            if (c < -1 || c > 1) {
                err = "coefficient outside {-1,0,1}";
                return -LCMA_ERR_COEFF_RANGE;
            }
    std::string first;
    if (scheme_brent_failures(s, &first) != 0) {
        err = first;
        return -LCMA_ERR_SCHEME_INVALID;
    }
    Registry& R = reg();
    std::lock_guard<std::mutex> g(R.mu);
    if (R.all.size() >= 256) {
        err = "scheme registry full";
        return -LCMA_ERR_NOT_SUPPORTED;
    }
    R.all.push_back(s);
    R.all.back().id = (int)R.all.size() - 1;
    return (int)R.all.size() - 1;
}

int scheme_parse(const std::string& text, Scheme& out, std::string& err) {
    std::istringstream in(text);
    std::string raw;
    std::vector<std::pair<int, std::string>> lines;
    int ln = 0;
    while (std::getline(in, raw)) {
        ++ln;
        auto h = raw.find('#');
        if (h != std::string::npos) raw = raw.substr(0, h);
        size_t a = raw.find_first_not_of(" \t\r");
        if (a == std::string::npos) continue;
        size_t b = raw.find_last_not_of(" \t\r");
        lines.emplace_back(ln, raw.substr(a, b - a + 1));
    }
    auto fail = [&](int line, const std::string& msg) {
        err = "line " + std::to_string(line) + ": " + msg;
        return -LCMA_ERR_PARSE;
    };
    if (lines.empty()) { err = "empty scheme file"; return -LCMA_ERR_PARSE; }
    {
        std::istringstream h(lines[0].second);
        if (!(h >> out.m >> out.k >> out.n >> out.R)) return fail(lines[0].first, "expected 'm k n R'");
        std::string extra;
        if (h >> extra) return fail(lines[0].first, "expected 'm k n R'");
    }
    if (out.m < 1 || out.k < 1 || out.n < 1 || out.R < 1 || out.R > 4096 || out.m > 16 ||
        out.k > 16 || out.n > 16)
        return fail(lines[0].first, "bad dimensions");
    size_t pos = 1;
    const char tags[3] = {'U', 'V', 'W'};
    const int rows_of[3] = {out.m, out.k, out.m}, cols_of[3] = {out.k, out.n, out.n};
    std::vector<int8_t>* T[3] = {&out.U, &out.V, &out.W};
    for (int t = 0; t < 3; ++t) {
        T[t]->assign((size_t)out.R * rows_of[t] * cols_of[t], 0);
        for (int r = 0; r < out.R; ++r) {
            if (pos >= lines.size()) { err = "unexpected end of file"; return -LCMA_ERR_PARSE; }
            std::istringstream h(lines[pos].second);
            std::string tag;
            int idx = -1;
            if (!(h >> tag >> idx) || tag.size() != 1 || tag[0] != tags[t] || idx != r + 1)
                return fail(lines[pos].first, std::string("expected '") + tags[t] + " " +
                                                  std::to_string(r + 1) + "'");
            ++pos;
            for (int i = 0; i < rows_of[t]; ++i) {
                if (pos >= lines.size()) { err = "unexpected end of file"; return -LCMA_ERR_PARSE; }
                std::istringstream rowin(lines[pos].second);
                for (int j = 0; j < cols_of[t]; ++j) {
                    long v;
                    if (!(rowin >> v)) return fail(lines[pos].first, "expected " + std::to_string(cols_of[t]) + " entries");
                    if (v < -1 || v > 1) {
                        err = "line " + std::to_string(lines[pos].first) + ": coefficient " +
                              std::to_string(v) + " outside {-1,0,1}";
                        return -LCMA_ERR_COEFF_RANGE;
                    }
                    (*T[t])[((size_t)r * rows_of[t] + i) * cols_of[t] + j] = (int8_t)v;
                }
                std::string extra;
                if (rowin >> extra) return fail(lines[pos].first, "too many entries");
                ++pos;
            }
        }
    }
    if (pos != lines.size()) return fail(lines[pos].first, "trailing content");
    return 0;
}

}  // namespace lcma

// ------------------------------------------------------------ product order
namespace lcma {
namespace {

struct OrderCost {
    int max_live;
    long long total_live;
    bool operator<(const OrderCost& o) const {
        return max_live != o.max_live ? max_live < o.max_live : total_live < o.total_live;
    }
};

// Live range of C_ij = [first position contributing, last position
// contributing).  A partial must be stored across the boundary after
// position t iff first <= t < last: the last contribution is consumed
// straight into the rounded C store, and a home freed by it can take a first
// contribution of the same product (the epilogue handles last contributions
// first, element by element in the same thread).
OrderCost order_cost(const Scheme& s, const std::vector<int>& perm) {
    const int mn = s.m * s.n, R = s.R;
    std::vector<int> first(mn, -1), last(mn, -1);
    for (int t = 0; t < R; ++t)
        for (int ij = 0; ij < mn; ++ij)
            if (s.W[(size_t)perm[t] * mn + ij]) {
                if (first[ij] < 0) first[ij] = t;
                last[ij] = t;
            }
    OrderCost c{0, 0};
    for (int t = 0; t < R; ++t) {
        int live = 0;
        for (int ij = 0; ij < mn; ++ij) live += (first[ij] >= 0 && first[ij] <= t && t < last[ij]);
        c.max_live = std::max(c.max_live, live);
        c.total_live += live;
    }
    return c;
}

ProductOrder compute_order(const Scheme& s) {
    const int R = s.R, mn = s.m * s.n;
    std::vector<int> best(R);
    for (int r = 0; r < R; ++r) best[r] = r;
    OrderCost best_c = order_cost(s, best);
    if (R <= 8) {
        std::vector<int> p = best;
        std::sort(p.begin(), p.end());
        do {
            OrderCost c = order_cost(s, p);
            if (c < best_c) { best_c = c; best = p; }
        } while (std::next_permutation(p.begin(), p.end()));
    } else {
        // deterministic restarts (LCG) + first-improvement pairwise-swap descent
        unsigned long long st = 0x9E3779B97F4A7C15ull;
        for (int restart = 0; restart < 24; ++restart) {
            std::vector<int> p(R);
            for (int r = 0; r < R; ++r) p[r] = r;
            if (restart > 0)
                for (int r = R - 1; r > 0; --r) {
                    st = st * 6364136223846793005ull + 1442695040888963407ull;
                    std::swap(p[r], p[(int)((st >> 33) % (unsigned long long)(r + 1))]);
                }
            OrderCost c = order_cost(s, p);
            bool improved = true;
            for (int pass = 0; improved && pass < 8; ++pass) {
                improved = false;
                for (int a = 0; a < R; ++a)
                    for (int b = a + 1; b < R; ++b) {
                        std::swap(p[a], p[b]);
                        OrderCost c2 = order_cost(s, p);
                        if (c2 < c) { c = c2; improved = true; }
                        else std::swap(p[a], p[b]);
                    }
            }
            if (c < best_c) { best_c = c; best = p; }
        }
    }
    ProductOrder o;
    o.perm = best;
    o.max_live = best_c.max_live;
    // interval colouring: C blocks in order of first use take the lowest slot
    // whose previous occupant's last use is not later than this first use
    std::vector<int> first(mn, -1), last(mn, -1), uses(mn, 0);
    for (int t = 0; t < R; ++t)
        for (int ij = 0; ij < mn; ++ij)
            if (s.W[(size_t)best[t] * mn + ij]) {
                if (first[ij] < 0) first[ij] = t;
                last[ij] = t;
                ++uses[ij];
            }
    std::vector<int> idx(mn);
    for (int ij = 0; ij < mn; ++ij) idx[ij] = ij;
    std::stable_sort(idx.begin(), idx.end(), [&](int a, int b) { return first[a] < first[b]; });
    o.slot.assign(mn, -1);
    std::vector<int> slot_end;   // last use of the current occupant of each slot
    for (int ij : idx) {
        if (first[ij] < 0) continue;
        if (first[ij] == last[ij]) { o.slot[ij] = -1; continue; }   // single contribution: no partial
        int chosen = -1;
        for (int sl = 0; sl < (int)slot_end.size(); ++sl)
            if (slot_end[sl] <= first[ij]) { chosen = sl; break; }
        if (chosen < 0) {
            chosen = (int)slot_end.size();
            slot_end.push_back(-1);
            o.slot_updates.push_back(0);
            o.slot_access.push_back(0);
        }
        slot_end[chosen] = last[ij];
        o.slot_updates[chosen] += uses[ij] - 1;   // stored partial accesses (all but the first's store)
        o.slot_access[chosen] += uses[ij];        // tile transfers if the slot lived in L2
        o.slot[ij] = chosen;
    }
    // home ranking: most-updated slots first (registers, then shared memory)
    const int ns = (int)slot_end.size();
    o.by_use.resize(ns);
    for (int k = 0; k < ns; ++k) o.by_use[k] = k;
    std::stable_sort(o.by_use.begin(), o.by_use.end(),
                     [&](int a, int b) { return o.slot_updates[a] > o.slot_updates[b]; });
    o.l2_tiles = 0.0;
    for (int k = 0; k < ns; ++k)
        o.l2_tiles += k == 0 ? 0.0 : k == 1 ? 0.5 * o.slot_access[o.by_use[k]] : (double)o.slot_access[o.by_use[k]];
    o.nslot = (int)slot_end.size();
    return o;
}

}  // namespace

const ProductOrder& scheme_product_order(int id) {
    static std::mutex mu;
    static std::vector<std::unique_ptr<ProductOrder>> cache(256);
    std::lock_guard<std::mutex> g(mu);
    if (id < 0 || id >= 256) id = 0;
    if (!cache[id]) {
        const Scheme* s = scheme_get(id);
        cache[id].reset(new ProductOrder(compute_order(*s)));
    }
    return *cache[id];
}

}  // namespace lcma
