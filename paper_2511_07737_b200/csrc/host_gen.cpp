// host_gen.cpp - native instance generators, DIMACS writer and model checker
// (§8(d) "Generators. Host C++, deterministic from
// seed"; SPEC S:50-58 verify_model).  Host-only C-ABI (include/turbosat.h).
//
// * planted random k-SAT (§8(d) "planted-k-SAT (naive)"): sigma uniform; each
//   clause draws k distinct variables uniformly (rejection of repeats); the
//   clause's truth pattern under sigma is uniform over the 2^k - 1 non-zero
//   patterns (hidden = 1), or over 1 .. 2^k - 2 so that the complement of
//   sigma satisfies it too (hidden = 2, "2-hidden" planting);
// * industrial-shaped CNF (§8(d)): clause lengths i.i.d. from a given
//   distribution, variables drawn with probability proportional to
//   rank^-alpha under a random id permutation (the scale-free structure of
//   industrial instances the paper cites), k distinct per
//   clause, signs planted as above;
// * DIMACS text writer (the planted model as a comment for V <= 64);
// * verify_model: number of clauses a 0/1 assignment leaves unsatisfied.
//
// The random stream is SplitMix64 (Steele et al., 2014) seeded from (seed,
// kind, V, C, k): deterministic per seed, documented, independent of the
// Python generators in tsat_synth/ (which the parity tests use).
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <new>
#include <string>
#include <vector>

#include "turbosat.h"

namespace {

struct SplitMix64 {
    uint64_t s;
    uint64_t next() {
        uint64_t z = (s += 0x9E3779B97F4A7C15ull);
        z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
        z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
        return z ^ (z >> 31);
    }
    // uniform in [0, n) without modulo bias (Lemire's multiply-shift with rejection)
    uint64_t below(uint64_t n) {
        for (;;) {
            const uint64_t x = next();
            const unsigned __int128 m = (unsigned __int128)x * n;
            const uint64_t lo = (uint64_t)m;
            if (lo >= n || lo >= (0 - n) % n) return (uint64_t)(m >> 64);
        }
    }
    double unit() { return (double)(next() >> 11) * 0x1.0p-53; }   // [0, 1)
};

uint64_t mix_seed(uint64_t seed, uint64_t kind, uint64_t V, uint64_t C, uint64_t k) {
    SplitMix64 r{seed ^ (kind * 0xD1B54A32D192ED03ull)};
    uint64_t h = r.next();
    for (uint64_t x : {V, C, k}) {
        r.s ^= x + 0x632BE59BD9B4E019ull + (h << 6) + (h >> 2);
        h = r.next();
    }
    return h;
}

// k distinct variables (rejection of repeats), then signs planted under sigma.
template <typename Draw>
void make_clause(SplitMix64& rng, Draw draw, int k, const std::vector<uint8_t>& sigma, int hidden, int32_t* out) {
    for (;;) {
        for (int i = 0; i < k; ++i) out[i] = (int32_t)draw();
        bool ok = true;
        for (int i = 1; i < k && ok; ++i)
            for (int j = 0; j < i; ++j)
                if (out[i] == out[j]) { ok = false; break; }
        if (ok) break;
    }
    // truth pattern t: bit i set <=> literal i is true under sigma
    const uint64_t npat = (k >= 63) ? ~0ull : ((1ull << k) - (hidden == 2 ? 2 : 1));
    const uint64_t t = 1 + rng.below(npat);
    for (int i = 0; i < k; ++i) {
        const int v = out[i];                                  // 0-based
        const bool truth = (t >> i) & 1ull;
        const bool pos = truth == (sigma[v] != 0);             // positive literal true iff sigma_v = 1
        out[i] = pos ? v + 1 : -(v + 1);
    }
}

}  // namespace

extern "C" tsat_status tsat_gen_planted(int32_t V, int64_t C, int32_t k, uint64_t seed, int32_t hidden,
                                        int64_t* clause_ptr, int32_t* dimacs_lits, uint8_t* sigma) {
    if (V < 1 || C < 0 || k < 1 || k > 15 || k > V || (hidden != 1 && hidden != 2) || (hidden == 2 && k < 2) ||
        !clause_ptr || (C > 0 && !dimacs_lits) || !sigma)
        return TSAT_E_ARG;
    try {
        SplitMix64 rng{mix_seed(seed, hidden == 2 ? 0x2A : 0x7A7, (uint64_t)V, (uint64_t)C, (uint64_t)k)};
        std::vector<uint8_t> sg((size_t)V);
        for (int32_t v = 0; v < V; ++v) sg[v] = (uint8_t)(rng.next() >> 63);
        auto draw = [&]() { return (int32_t)rng.below((uint64_t)V); };
        for (int64_t c = 0; c <= C; ++c) clause_ptr[c] = c * k;
        for (int64_t c = 0; c < C; ++c) make_clause(rng, draw, k, sg, hidden, dimacs_lits + c * k);
        std::memcpy(sigma, sg.data(), (size_t)V);
        return TSAT_OK;
    } catch (const std::bad_alloc&) {
        return TSAT_E_OOM;
    }
}

extern "C" tsat_status tsat_gen_industrial(int32_t V, int64_t C, uint64_t seed, double alpha, int32_t kmax,
                                           const double* len_probs, int64_t* clause_ptr, int32_t* dimacs_lits,
                                           int64_t lits_capacity, uint8_t* sigma) {
    if (V < 1 || C < 0 || kmax < 1 || kmax > 15 || kmax > V || !len_probs || !clause_ptr || !sigma || !(alpha >= 0) ||
        (C > 0 && (!dimacs_lits || lits_capacity < C * kmax)))
        return TSAT_E_ARG;
    double tot = 0.0;
    for (int i = 0; i <= kmax; ++i) {
        if (!(len_probs[i] >= 0)) return TSAT_E_ARG;
        tot += len_probs[i];
    }
    if (!(tot > 0) || len_probs[0] > 0) return TSAT_E_ARG;          // no empty clauses by construction
    try {
        SplitMix64 rng{mix_seed(seed, 0x1D5, (uint64_t)V, (uint64_t)C, (uint64_t)kmax)};
        std::vector<uint8_t> sg((size_t)V);
        for (int32_t v = 0; v < V; ++v) sg[v] = (uint8_t)(rng.next() >> 63);
        std::vector<double> lcdf((size_t)kmax + 1);
        double acc = 0.0;
        for (int i = 0; i <= kmax; ++i) { acc += len_probs[i] / tot; lcdf[i] = acc; }
        // variable weights rank^-alpha over a random permutation of the ids
        std::vector<double> cdf((size_t)V);
        acc = 0.0;
        for (int32_t r = 0; r < V; ++r) { acc += std::pow((double)(r + 1), -alpha); cdf[r] = acc; }
        for (double& x : cdf) x /= acc;
        std::vector<int32_t> perm((size_t)V);
        for (int32_t v = 0; v < V; ++v) perm[v] = v;
        for (int32_t i = V - 1; i > 0; --i) std::swap(perm[i], perm[(size_t)rng.below((uint64_t)i + 1)]);
        auto draw = [&]() {
            const double u = rng.unit();
            size_t r = (size_t)(std::upper_bound(cdf.begin(), cdf.end(), u) - cdf.begin());
            if (r >= (size_t)V) r = (size_t)V - 1;
            return perm[r];
        };
        int64_t p = 0;
        clause_ptr[0] = 0;
        for (int64_t c = 0; c < C; ++c) {
            const double u = rng.unit();
            int k = (int)(std::upper_bound(lcdf.begin(), lcdf.end(), u) - lcdf.begin());
            if (k > kmax) k = kmax;
            if (k < 1) k = 1;
            make_clause(rng, draw, k, sg, 1, dimacs_lits + p);
            p += k;
            clause_ptr[c + 1] = p;
        }
        std::memcpy(sigma, sg.data(), (size_t)V);
        return TSAT_OK;
    } catch (const std::bad_alloc&) {
        return TSAT_E_OOM;
    }
}

extern "C" tsat_status tsat_write_dimacs(int32_t V, int64_t C, const int64_t* clause_ptr, const int32_t* dimacs_lits,
                                         const uint8_t* sigma, char* out, size_t capacity, size_t* length) {
    if (V < 0 || C < 0 || !clause_ptr || (C > 0 && !dimacs_lits) || !length) return TSAT_E_ARG;
    for (int64_t c = 0; c < C; ++c)
        if (clause_ptr[c + 1] < clause_ptr[c]) return TSAT_E_ARG;
    try {
        std::string s;
        s.reserve((size_t)(C > 0 ? clause_ptr[C] - clause_ptr[0] : 0) * 8 + 64);
        if (sigma && V <= 64) {
            s += "c planted";
            for (int32_t v = 0; v < V; ++v) { s += ' '; s += (char)('0' + (sigma[v] ? 1 : 0)); }
            s += '\n';
        }
        char buf[64];
        std::snprintf(buf, sizeof buf, "p cnf %d %lld\n", V, (long long)C);
        s += buf;
        for (int64_t c = 0; c < C; ++c) {
            for (int64_t j = clause_ptr[c]; j < clause_ptr[c + 1]; ++j) {
                if (dimacs_lits[j] == 0 || std::abs(dimacs_lits[j]) > V) return TSAT_E_ARG;
                s += std::to_string(dimacs_lits[j]);
                s += ' ';
            }
            s += "0\n";
        }
        *length = s.size();
        if (!out) return TSAT_OK;                                      // size query
        if (capacity < s.size()) return TSAT_E_RANGE;
        std::memcpy(out, s.data(), s.size());
        return TSAT_OK;
    } catch (const std::bad_alloc&) {
        return TSAT_E_OOM;
    }
}

extern "C" tsat_status tsat_verify_model(int32_t V, int64_t C, const int64_t* clause_ptr, const int32_t* dimacs_lits,
                                         const uint8_t* model, int64_t* n_unsat) {
    if (V < 0 || C < 0 || !clause_ptr || (C > 0 && !dimacs_lits) || !model || !n_unsat) return TSAT_E_ARG;
    int64_t bad = 0;
    for (int64_t c = 0; c < C; ++c) {
        if (clause_ptr[c + 1] < clause_ptr[c]) return TSAT_E_ARG;
        bool sat = false;
        for (int64_t j = clause_ptr[c]; j < clause_ptr[c + 1]; ++j) {
            const int32_t x = dimacs_lits[j];
            if (x == 0 || std::abs(x) > V) return TSAT_E_ARG;
            if ((model[std::abs(x) - 1] != 0) == (x > 0)) { sat = true; break; }
        }
        bad += sat ? 0 : 1;
    }
    *n_unsat = bad;
    return TSAT_OK;
}
