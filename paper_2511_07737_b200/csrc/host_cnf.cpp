// host_cnf.cpp - DIMACS parser and the clause store (CSR clause->literal plus
// its transpose variable->occurrence), host side.
//
// DIMACS conventions follow SPEC.md S:41-49: comment lines 'c', header
// 'p cnf V C', clauses of signed integers terminated by 0; header/body
// clause-count mismatch is a warning; duplicate literals are removed;
// tautologies are kept (counted); empty clauses are preserved; errors for a
// malformed header, '-0', a variable > V, or a non-integer token.
#include <algorithm>
#include <cstring>
#include <string>
#include <vector>

#include "tsat_internal.h"

namespace tsat {

namespace {

struct Lexer {
    const char* p;
    const char* end;
    int64_t line = 1;
    void skip_ws() {
        while (p < end && (*p == ' ' || *p == '\t' || *p == '\r' || *p == '\n' || *p == '\f' || *p == '\v')) {
            if (*p == '\n') ++line;
            ++p;
        }
    }
    void skip_line() {
        while (p < end && *p != '\n') ++p;
    }
    // token [b, e)
    bool token(const char** b, const char** e) {
        skip_ws();
        if (p >= end) return false;
        *b = p;
        while (p < end && !(*p == ' ' || *p == '\t' || *p == '\r' || *p == '\n' || *p == '\f' || *p == '\v')) ++p;
        *e = p;
        return true;
    }
};

bool parse_int(const char* b, const char* e, int64_t* out, bool* neg_zero) {
    *neg_zero = false;
    if (b == e) return false;
    bool neg = false;
    const char* q = b;
    if (*q == '-' || *q == '+') { neg = (*q == '-'); ++q; }
    if (q == e) return false;
    int64_t v = 0;
    for (; q < e; ++q) {
        if (*q < '0' || *q > '9') return false;
        v = v * 10 + (*q - '0');
        if (v > (int64_t)1 << 40) return false;
    }
    if (neg && v == 0) *neg_zero = true;
    *out = neg ? -v : v;
    return true;
}

}  // namespace

int parse_dimacs(const char* text, size_t len, int32_t* V_out, std::vector<int64_t>* ptr,
                 std::vector<int32_t>* lits, int64_t* header_C, int64_t* n_warnings, std::string* msg) {
    Lexer lx{text, text + len};
    int64_t V = -1, Chdr = -1;
    ptr->assign(1, 0);
    lits->clear();
    *n_warnings = 0;
    bool in_clause = false;
    while (true) {
        lx.skip_ws();
        if (lx.p >= lx.end) break;
        char ch = *lx.p;
        if (ch == 'c' && !in_clause) {          // comment line
            lx.skip_line();
            continue;
        }
        if (ch == '%' && !in_clause) {          // SATLIB end marker
            break;
        }
        if (ch == 'p') {
            if (V >= 0) { *msg = "duplicate header at line " + std::to_string(lx.line); return 2; }
            if (in_clause) { *msg = "header inside a clause at line " + std::to_string(lx.line); return 2; }
            const char *b, *e;
            lx.token(&b, &e);
            if (e - b != 1) { *msg = "malformed header at line " + std::to_string(lx.line); return 2; }
            if (!lx.token(&b, &e) || (e - b) != 3 || std::strncmp(b, "cnf", 3) != 0) {
                *msg = "malformed header (expected 'p cnf V C') at line " + std::to_string(lx.line);
                return 2;
            }
            bool nz;
            if (!lx.token(&b, &e) || !parse_int(b, e, &V, &nz) || V < 0 || V > (1 << 29)) {
                *msg = "malformed header: bad variable count at line " + std::to_string(lx.line);
                return 2;
            }
            if (!lx.token(&b, &e) || !parse_int(b, e, &Chdr, &nz) || Chdr < 0) {
                *msg = "malformed header: bad clause count at line " + std::to_string(lx.line);
                return 2;
            }
            continue;
        }
        const char *b, *e;
        lx.token(&b, &e);
        int64_t x;
        bool negzero;
        if (!parse_int(b, e, &x, &negzero)) {
            *msg = "non-integer token '" + std::string(b, std::min<size_t>(e - b, 32)) + "' at line " + std::to_string(lx.line);
            return 2;
        }
        if (V < 0) { *msg = "clause before the 'p cnf' header at line " + std::to_string(lx.line); return 2; }
        if (negzero) { *msg = "literal -0 inside a clause at line " + std::to_string(lx.line); return 2; }
        if (x == 0) {
            ptr->push_back((int64_t)lits->size());
            in_clause = false;
            continue;
        }
        int64_t a = x < 0 ? -x : x;
        if (a > V) {
            *msg = "variable " + std::to_string(a) + " > V=" + std::to_string(V) + " at line " + std::to_string(lx.line);
            return 2;
        }
        lits->push_back((int32_t)x);
        in_clause = true;
    }
    if (V < 0) { *msg = "missing 'p cnf V C' header"; return 2; }
    if (in_clause) {                          // last clause without its terminating 0
        ptr->push_back((int64_t)lits->size());
        ++*n_warnings;
    }
    int64_t C = (int64_t)ptr->size() - 1;
    if (C != Chdr) ++*n_warnings;
    *V_out = (int32_t)V;
    *header_C = Chdr;
    return 0;
}

// Batched occurrence records (k_update's general gather): per row and sign
// section (negated first), the records sorted by clause length, longest first
// (stable; the counts do not depend on the order, R12), cut into batches of
// 4.  A batch is a header word (J << 4) | (count << 1) | negated, count =
// records in the batch (1..4), J = longest length - 1, then J x 4 literal
// codes [j][k] = the (j+1)-th other literal of record k, or the padding code
// V << 1 (row V of each bit-plane buffer is all zero, so it adds nothing) for
// a shorter or absent record.  The 4 records' gathers of one j are
// independent, and one batch is one carry-save sum4 per bin.
static void build_batched(HostCnf* hp) {
    HostCnf& h = *hp;
    const int32_t V = h.V;
    const uint32_t pad = (uint32_t)V << 1;
    h.bat_ptr.assign((size_t)V + 1, 0);
    h.bat_rec.clear();
    std::vector<uint32_t> sec;
    for (int32_t v = 0; v < V; ++v) {
        h.bat_ptr[v] = (uint32_t)h.bat_rec.size();
        const uint32_t b = h.occ_ptr[v], e = h.occ_ptr[v + 1];
        for (int sidx = 0; sidx < 2; ++sidx) {
            const uint32_t neg = 1 - sidx;                       // negated section, then positive
            sec.clear();
            for (uint32_t p = b; p < e; p += h.occ_rec[p] >> 1)
                if ((h.occ_rec[p] & 1u) == neg) sec.push_back(p);
            std::stable_sort(sec.begin(), sec.end(),
                             [&](uint32_t x, uint32_t y) { return (h.occ_rec[x] >> 1) > (h.occ_rec[y] >> 1); });
            for (size_t i = 0; i < sec.size(); i += 4) {
                const uint32_t cnt = (uint32_t)std::min<size_t>(4, sec.size() - i);
                const uint32_t J = (h.occ_rec[sec[i]] >> 1) - 1;
                h.bat_rec.push_back((J << 4) | (cnt << 1) | neg);
                for (uint32_t j = 0; j < J; ++j)
                    for (uint32_t k = 0; k < 4; ++k) {
                        uint32_t code = pad;
                        if (k < cnt) {
                            const uint32_t p = sec[i + k];
                            if (j + 1 < (h.occ_rec[p] >> 1)) code = h.occ_rec[p + 1 + j];
                        }
                        h.bat_rec.push_back(code);
                    }
            }
        }
    }
    h.bat_ptr[V] = (uint32_t)h.bat_rec.size();
}

// Length segments for k_clause_seg (K <= 7): the clauses regrouped by length
// L = 1..7, each segment a dense [C_L][L] array of literal codes, so a warp
// evaluates exactly L literals and L + 1 bins per clause instead of padding
// every clause to K.  Empty clauses join the L = 1 segment as the literal
// "row V" (the all-zero plane: always false, R = 0).  The histogram counts do
// not depend on clause order (R12).
static void build_segments(HostCnf* hp) {
    HostCnf& h = *hp;
    h.seg_C.assign(8, 0);
    h.seg_off.assign(8, 0);
    h.seg_lit.clear();
    if (h.K > 7) return;
    for (int64_t c = 0; c < h.C; ++c) {
        const uint32_t len = h.clause_ptr[c + 1] - h.clause_ptr[c];
        h.seg_C[len == 0 ? 1 : len] += 1;
    }
    int64_t off = 0;
    for (int L = 1; L <= 7; ++L) { h.seg_off[L] = off; off += h.seg_C[L] * L; }
    h.seg_lit.assign((size_t)off, 0);
    std::vector<int64_t> fill(h.seg_off.begin(), h.seg_off.end());
    for (int64_t c = 0; c < h.C; ++c) {
        const uint32_t b = h.clause_ptr[c], e = h.clause_ptr[c + 1];
        if (b == e) { h.seg_lit[(size_t)fill[1]++] = (uint32_t)h.V << 1; continue; }
        int64_t& f = fill[e - b];
        for (uint32_t i = b; i < e; ++i) h.seg_lit[(size_t)f++] = h.clause_lit[i];
    }
}

// bat_rec offsets are stored as uint32 (bat_ptr, hub super-chunks)
static bool batched_fits(const HostCnf& h) { return h.bat_rec.size() < ((size_t)1 << 31); }

int build_cnf(int32_t V, int64_t C, const int64_t* ptr, const int32_t* lits, HostCnf* out, std::string* msg) {
    if (V < 0 || C < 0 || (C > 0 && (!ptr || (!lits && ptr[C] > 0)))) { *msg = "bad CNF arrays"; return 1; }
    if (V >= (1 << 29)) { *msg = "V too large (>= 2^29)"; return 3; }
    if (C > 0 && ptr[0] != 0) { *msg = "clause_ptr[0] must be 0"; return 1; }
    for (int64_t c = 0; c < C; ++c)
        if (ptr[c + 1] < ptr[c]) { *msg = "clause_ptr not monotone"; return 1; }
    if (C > 0 && ptr[C] >= ((int64_t)1 << 32)) { *msg = "too many literals (>= 2^32)"; return 3; }
    HostCnf h;
    h.V = V;
    h.C = C;
    h.clause_ptr.resize((size_t)C + 1);
    h.clause_ptr[0] = 0;
    std::vector<uint32_t> codes;
    codes.reserve(C > 0 ? (size_t)(ptr[C] - ptr[0]) : 0);
    // per-variable (clause stamp, mask of signs seen in that clause): O(nnz) dedup
    std::vector<int64_t> seen_stamp((size_t)V + 1, -1);
    std::vector<uint8_t> seen_mask((size_t)V + 1, 0);
    for (int64_t c = 0; c < C; ++c) {
        if (ptr[c + 1] < ptr[c]) { *msg = "clause_ptr not monotone"; return 1; }
        bool taut = false;
        size_t start = codes.size();
        for (int64_t l = ptr[c]; l < ptr[c + 1]; ++l) {
            int32_t x = lits[l];
            int64_t a = x < 0 ? -(int64_t)x : x;
            if (x == 0 || a > V) { *msg = "literal out of range in clause " + std::to_string(c); return 1; }
            uint8_t bit = x > 0 ? 1 : 2;
            if (seen_stamp[a] != c) { seen_stamp[a] = c; seen_mask[a] = 0; }
            if (seen_mask[a] & bit) { ++h.n_duplicates; continue; }
            if (seen_mask[a]) taut = true;
            seen_mask[a] |= bit;
            codes.push_back(((uint32_t)(a - 1) << 1) | (x < 0 ? 1u : 0u));
        }
        size_t len = codes.size() - start;
        if (len == 0) h.has_empty = 1;
        if (taut) ++h.n_tautologies;
        if ((int64_t)len > h.K) h.K = (int32_t)len;
        if (codes.size() > 0xffffffffull) { *msg = "too many literals (>= 2^32)"; return 3; }
        h.clause_ptr[(size_t)c + 1] = (uint32_t)codes.size();
    }
    h.nnz = (int64_t)codes.size();
    h.clause_lit.swap(codes);
    if (h.K > kMaxK) {
        *msg = "clause length " + std::to_string(h.K) + " > " + std::to_string(kMaxK) + " not supported";
        return 3;
    }
    // transpose: occurrence records per variable, clause-ascending
    h.occ_cnt.assign((size_t)V, 0);
    std::vector<uint64_t> words((size_t)V, 0);
    for (int64_t c = 0; c < C; ++c) {
        uint32_t len = h.clause_ptr[c + 1] - h.clause_ptr[c];
        for (uint32_t i = h.clause_ptr[c]; i < h.clause_ptr[c + 1]; ++i) {
            uint32_t v = h.clause_lit[i] >> 1;
            h.occ_cnt[v] += 1;
            words[v] += len;
        }
    }
    h.occ_ptr.assign((size_t)V + 1, 0);
    uint64_t acc = 0;
    for (int32_t v = 0; v < V; ++v) {
        h.occ_ptr[v] = (uint32_t)acc;
        acc += words[v];
        if (acc > 0xffffffffull) { *msg = "occurrence records too large (>= 2^32 words)"; return 3; }
    }
    h.occ_ptr[V] = (uint32_t)acc;
    h.occ_rec.assign(acc, 0);
    // records of negated occurrences first, then positive ones, each in clause
    // order: the kernels sum runs of same-sign occurrences with carry-save
    // adders (the counts do not depend on the order, R12)
    std::vector<uint64_t> negw((size_t)V, 0);
    for (int64_t c = 0; c < C; ++c) {
        uint32_t len = h.clause_ptr[c + 1] - h.clause_ptr[c];
        for (uint32_t i = h.clause_ptr[c]; i < h.clause_ptr[c + 1]; ++i)
            if (h.clause_lit[i] & 1u) negw[h.clause_lit[i] >> 1] += len;
    }
    std::vector<uint32_t> fill_neg(h.occ_ptr.begin(), h.occ_ptr.end() - 1), fill_pos((size_t)V);
    for (int32_t v = 0; v < V; ++v) fill_pos[v] = h.occ_ptr[v] + (uint32_t)negw[v];
    for (int64_t c = 0; c < C; ++c) {
        uint32_t b = h.clause_ptr[c], e = h.clause_ptr[c + 1], len = e - b;
        for (uint32_t i = b; i < e; ++i) {
            uint32_t code = h.clause_lit[i];
            uint32_t v = code >> 1;
            uint32_t& f = (code & 1u) ? fill_neg[v] : fill_pos[v];
            uint32_t* r = &h.occ_rec[f];
            r[0] = (len << 1) | (code & 1u);
            uint32_t o = 1;
            for (uint32_t j = b; j < e; ++j)
                if (j != i) r[o++] = h.clause_lit[j];
            f += len;
        }
    }
    // signed-count classes and hub super-chunks (see tsat_internal.h)
    h.occ_pn.assign((size_t)V * 2, 0);
    for (int64_t i = 0; i < h.nnz; ++i) {
        uint32_t code = h.clause_lit[i];
        h.occ_pn[(size_t)(code >> 1) * 2 + (code & 1u)] += 1;
    }
    h.uniform_len = 1;
    for (int64_t c = 0; c < C; ++c)
        if ((int32_t)(h.clause_ptr[c + 1] - h.clause_ptr[c]) != h.K) { h.uniform_len = 0; break; }
    // k_update stages uniform 3-SAT rows as plain records, every other
    // instance as batched records (build_batched)
    h.batched = !(h.uniform_len && h.K == 3);
    if (h.batched) {
        build_batched(&h);
        if (!batched_fits(h)) { *msg = "batched occurrence records too large (>= 2^31 words)"; return 3; }
    }
    const std::vector<uint32_t>& sptr = h.batched ? h.bat_ptr : h.occ_ptr;
    h.hub_of.assign((size_t)V, -1);
    for (int32_t v = 0; v < V; ++v) {
        const uint32_t staged = sptr[v + 1] - sptr[v];
        // K > 7 (KB = 16): every row's 15 bins are counted by k_hub (int32)
        bool hub = h.K > 7 || h.occ_pn[2 * v] > 127 || h.occ_pn[2 * v + 1] > 127 || (h.occ_ptr[v + 1] - h.occ_ptr[v]) > (uint32_t)kRecCap ||
                   staged > (uint32_t)kRecCap;
        if (!hub) {
            h.max_rec_words = std::max<int32_t>(h.max_rec_words, (int32_t)staged);
            continue;
        }
        int32_t hid = h.n_hubs++;
        h.hub_of[v] = hid;
        if (h.batched) {                 // super-chunks of kHubSlabBatches batched-record batches
            uint32_t p = h.bat_ptr[v], e = h.bat_ptr[v + 1], b = p;
            int cnt = 0;
            while (p < e) {
                p += 1 + 4 * (h.bat_rec[p] >> 4);
                if (++cnt == kHubSlabBatches || p >= e) {
                    h.hub_sc.insert(h.hub_sc.end(), {hid, v, (int32_t)b, (int32_t)p});
                    b = p;
                    cnt = 0;
                }
            }
            continue;
        }
        uint32_t p = h.occ_ptr[v], e = h.occ_ptr[v + 1], b = p;
        int cnt = 0;
        while (p < e) {
            p += h.occ_rec[p] >> 1;
            if (++cnt == kHubSlab || p >= e) {
                h.hub_sc.insert(h.hub_sc.end(), {hid, v, (int32_t)b, (int32_t)p});
                b = p;
                cnt = 0;
            }
        }
    }
    h.n_hub_sc = (int32_t)(h.hub_sc.size() / 4);
    build_segments(&h);
    *out = std::move(h);
    return 0;
}

}  // namespace tsat
