// schemes.h -- LCMA scheme registry of the product library (host).
// An LCMA is the tuple <m,k,n,R,U,V,W>; U[r][i][l] multiplies
// A_{i,l} (Eq. 3), V[r][l][j] multiplies B_{l,j} (Eq. 4), W[r][i][j] adds H_r
// into C_{i,j} (Eq. 6).  Coefficients restricted to {-1,0,1}.
#pragma once
#include <stdint.h>

#include <string>
#include <vector>

namespace lcma {

struct Scheme {
    std::string name;
    int id = -1;                   // registry id (set on registration)
    int base_id = -1;              // >= 0: this scheme is compose(base, base)
    int m = 1, k = 1, n = 1, R = 1;
    std::vector<int8_t> U, V, W;   // R*m*k, R*k*n, R*m*n
    int8_t u(int r, int i, int l) const { return U[(r * m + i) * k + l]; }
    int8_t v(int r, int l, int j) const { return V[(r * k + l) * n + j]; }
    int8_t w(int r, int i, int j) const { return W[(r * m + i) * n + j]; }
    int nnzU() const;
    int nnzV() const;
    int nnzW() const;
};

// Built-in ids: 0 classical <1,1,1;1>, 1 Strassen, 2 Strassen^2, 3 Laderman.
enum : int { SCHEME_CLASSICAL = 0, SCHEME_STRASSEN = 1, SCHEME_STRASSEN2 = 2, SCHEME_LADERMAN = 3 };

// Returns nullptr for an unknown id.  Thread-safe.
const Scheme* scheme_get(int id);
// Validates (Brent identity, coefficient range, size limits) and registers.
// On failure returns a negative lcma_status and fills `err`.
int scheme_register(const Scheme& s, std::string& err);
// Text format of SPEC S:143-145.
int scheme_parse(const std::string& text, Scheme& out, std::string& err);
// Exact Brent check; returns number of failing tuples, first failure in `err`.
long long scheme_brent_failures(const Scheme& s, std::string* first);
Scheme scheme_compose(const Scheme& outer, const Scheme& inner);

// Processing order of the R products inside a group for the fused Combine H
// epilogue, chosen to minimise the number of C_ij partial tiles live at the
// same time (then their total live length), and the resulting assignment of
// C_ij to shared partial slots (C blocks with disjoint live ranges share one).
struct ProductOrder {
    std::vector<int> perm;           // position t -> product r
    std::vector<int> slot;           // C_ij -> slot (-1: one contribution, never stored)
    std::vector<int> slot_updates;   // per slot: partial read-modify-writes over a group
    std::vector<int> slot_access;    // per slot: partial tile transfers over a group if homed in L2
    std::vector<int> by_use;         // slots by decreasing updates: [0] -> registers, [1] -> shared memory
    double l2_tiles = 0.0;           // partial tile transfers per group that still go to L2 (the
                                     // shared-memory home holds column half 0 only)
    int nslot = 0;                   // partials live at once (per CTA)
    int max_live = 0;
};
// Cached per scheme id; deterministic.
const ProductOrder& scheme_product_order(int id);

}  // namespace lcma
