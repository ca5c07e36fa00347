// host_cdcl.cpp - SURVEY §8(f) f1: the CPU side of TurboSAT's hand-off
// (§4.2 l.277-287).  "Each thread receives a partial initialization
// from the GPU and executes a CDCL-based SAT solver instance from the partial
// initialization" (l.283); the number of instances "scales with the number of
// CPU threads available" and, when threads are scarce, "we prioritize the
// assignments with higher number of satisfied clauses" (l.285-286).
//
// A compact conflict-driven clause-learning solver (two watched literals,
// first-UIP learning with local minimisation, VSIDS on a binary heap, phase
// saving, Luby restarts, activity-based learnt-clause reduction) plus a
// portfolio driver: the k confident literals of each exported candidate
// (tsat_export_best) are assumed as the first decisions ("assigning V*
// variables prunes the search space by 2^V*", l.291), so a seed that
// contradicts every model fails fast (UNSAT under assumptions) and the thread
// takes the next one.  One instance runs unseeded so the portfolio stays
// complete.  The first thread to find a model stops the others.
//
// Host-only; it is the consumer the export hook feeds, not part of the GPU
// step (the north star keeps CDCL out of the data-parallel hot path).
#include <algorithm>
#include <atomic>
#include <chrono>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <mutex>
#include <new>
#include <thread>
#include <vector>

#include "turbosat.h"

namespace tsat {
namespace cdcl {

enum : int { kUnknown = 0, kSat = 10, kUnsat = 20, kUnsatAssump = 21 };

struct Clause {
    std::vector<int> lits;     // lits[0], lits[1] watched
    double act = 0.0;
    bool learnt = false;
    bool dead = false;
};

class Solver {
public:
    Solver(int nv, uint64_t seed) : nv_(nv), rng_(seed * 0x9E3779B97F4A7C15ull + 1) {
        val_.assign(nv, -1);
        level_.assign(nv, 0);
        reason_.assign(nv, -1);
        act_.assign(nv, 0.0);
        phase_.assign(nv, 0);
        seen_.assign(nv, 0);
        watches_.resize(2 * (size_t)nv);
        heap_pos_.assign(nv, -1);
        if (seed) {        // portfolio diversity: tiny random activities, random initial phases
            for (int v = 0; v < nv; ++v) {
                act_[v] = 1e-6 * (double)(next() % 1000);
                phase_[v] = (int8_t)(next() & 1);
            }
        }
        for (int v = 0; v < nv; ++v) heap_insert(v);
    }

    // Adds an input clause (internal literals 2v | neg).  False: the formula
    // is trivially unsatisfiable (empty clause or conflicting units).
    bool add_clause(std::vector<int> c) {
        std::sort(c.begin(), c.end());
        c.erase(std::unique(c.begin(), c.end()), c.end());
        for (size_t i = 1; i < c.size(); ++i)
            if (c[i] == (c[i - 1] ^ 1)) return true;          // tautology
        if (c.empty()) { ok_ = false; return false; }
        if (c.size() == 1) {
            const int l = c[0];
            if (value(l) == 0) { ok_ = false; return false; }
            if (value(l) < 0) enqueue(l, -1);
            return true;
        }
        attach(add(std::move(c), false));
        return true;
    }

    // Solve under assumptions; stop is polled.  Returns kSat / kUnsat /
    // kUnsatAssump / kUnknown (limit or stop).
    int solve(const std::vector<int>& assumptions, int64_t conflict_limit, const std::atomic<int>* stop,
              std::chrono::steady_clock::time_point deadline) {
        if (!ok_) return kUnsat;
        if (propagate() >= 0) return kUnsat;
        assumptions_ = assumptions;
        max_learnts_ = std::max<double>(1000.0, (double)clauses_.size() / 3.0);
        int64_t restart_no = 0;
        for (;;) {
            const int64_t budget = (int64_t)(luby(2.0, restart_no++) * 100.0);
            const int r = search(budget, conflict_limit, stop, deadline);
            if (r != kUnknown || stopped_) return r;
            max_learnts_ *= 1.05;
        }
    }

    const std::vector<int8_t>& values() const { return val_; }
    int64_t conflicts = 0, decisions = 0, propagations = 0;

private:
    int nv_;
    uint64_t rng_;
    bool ok_ = true, stopped_ = false;
    std::vector<Clause> clauses_;
    struct Watch { int ci, blocker; };
    std::vector<std::vector<Watch>> watches_;   // literal -> clauses watching it (+ a blocker literal)
    std::vector<int8_t> val_, phase_, seen_;
    std::vector<int> level_, reason_, trail_, trail_lim_, assumptions_;
    std::vector<double> act_;
    std::vector<int> heap_, heap_pos_;
    std::vector<int> learnt_idx_;
    size_t qhead_ = 0;
    double var_inc_ = 1.0, cla_inc_ = 1.0, max_learnts_ = 0.0;

    uint64_t next() {
        rng_ ^= rng_ << 13; rng_ ^= rng_ >> 7; rng_ ^= rng_ << 17;
        return rng_;
    }
    static double luby(double y, int64_t x) {
        int64_t size = 1, seq = 0;
        while (size < x + 1) { ++seq; size = 2 * size + 1; }
        while (size - 1 != x) { size = (size - 1) >> 1; --seq; x = x % size; }
        return std::pow(y, (double)seq);
    }
    int value(int lit) const {                       // -1 undef, 0 false, 1 true
        const int8_t x = val_[lit >> 1];
        return x < 0 ? -1 : (x ^ (lit & 1));
    }
    int level() const { return (int)trail_lim_.size(); }
    int add(std::vector<int> c, bool learnt) {
        Clause cl;
        cl.lits = std::move(c);
        cl.learnt = learnt;
        clauses_.push_back(std::move(cl));
        return (int)clauses_.size() - 1;
    }
    void attach(int ci) {
        const Clause& c = clauses_[ci];
        watches_[c.lits[0]].push_back({ci, c.lits[1]});
        watches_[c.lits[1]].push_back({ci, c.lits[0]});
    }
    void enqueue(int lit, int reason) {
        const int v = lit >> 1;
        val_[v] = (int8_t)((lit & 1) ^ 1);
        level_[v] = level();
        reason_[v] = reason;
        trail_.push_back(lit);
    }
    // heap (max activity on top)
    bool less(int a, int b) const { return act_[a] > act_[b]; }
    void heap_up(int i) {
        const int v = heap_[i];
        while (i > 0) {
            const int p = (i - 1) >> 1;
            if (!less(v, heap_[p])) break;
            heap_[i] = heap_[p]; heap_pos_[heap_[i]] = i; i = p;
        }
        heap_[i] = v; heap_pos_[v] = i;
    }
    void heap_down(int i) {
        const int v = heap_[i], n = (int)heap_.size();
        for (;;) {
            int c = 2 * i + 1;
            if (c >= n) break;
            if (c + 1 < n && less(heap_[c + 1], heap_[c])) ++c;
            if (!less(heap_[c], v)) break;
            heap_[i] = heap_[c]; heap_pos_[heap_[i]] = i; i = c;
        }
        heap_[i] = v; heap_pos_[v] = i;
    }
    void heap_insert(int v) {
        if (heap_pos_[v] >= 0) return;
        heap_.push_back(v);
        heap_up((int)heap_.size() - 1);
    }
    int heap_pop() {
        const int v = heap_[0];
        heap_[0] = heap_.back();
        heap_.pop_back();
        heap_pos_[v] = -1;
        if (!heap_.empty()) { heap_pos_[heap_[0]] = 0; heap_down(0); }
        return v;
    }
    void bump_var(int v) {
        act_[v] += var_inc_;
        if (act_[v] > 1e100) {
            for (double& a : act_) a *= 1e-100;
            var_inc_ *= 1e-100;
        }
        if (heap_pos_[v] >= 0) heap_up(heap_pos_[v]);
    }
    void bump_clause(Clause& c) {
        c.act += cla_inc_;
        if (c.act > 1e20) {
            for (int i : learnt_idx_) clauses_[i].act *= 1e-20;
            cla_inc_ *= 1e-20;
        }
    }

    // Unit propagation; returns the conflicting clause or -1.
    int propagate() {
        int confl = -1;
        while (qhead_ < trail_.size()) {
            const int p = trail_[qhead_++];
            const int fl = p ^ 1;                                   // the literal that became false
            std::vector<Watch>& ws = watches_[fl];
            ++propagations;
            size_t i = 0, j = 0;
            while (i < ws.size()) {
                const Watch wch = ws[i++];
                if (value(wch.blocker) == 1) { ws[j++] = wch; continue; }   // satisfied: clause untouched
                const int ci = wch.ci;
                Clause& c = clauses_[ci];
                if (c.dead) continue;
                if (c.lits[0] == fl) std::swap(c.lits[0], c.lits[1]);
                if (value(c.lits[0]) == 1) { ws[j++] = {ci, c.lits[0]}; continue; }
                bool moved = false;
                for (size_t k = 2; k < c.lits.size(); ++k) {
                    if (value(c.lits[k]) != 0) {
                        std::swap(c.lits[1], c.lits[k]);
                        watches_[c.lits[1]].push_back({ci, c.lits[0]});
                        moved = true;
                        break;
                    }
                }
                if (moved) continue;
                ws[j++] = {ci, c.lits[0]};
                if (value(c.lits[0]) == 0) {                        // conflict: keep the remaining watches
                    confl = ci;
                    qhead_ = trail_.size();
                    while (i < ws.size()) ws[j++] = ws[i++];
                } else {
                    enqueue(c.lits[0], ci);
                }
            }
            ws.resize(j);
            if (confl >= 0) break;
        }
        return confl;
    }

    // First-UIP conflict analysis; out[0] is the asserting literal.
    void analyze(int confl, std::vector<int>& out, int& bt_level) {
        out.clear();
        out.push_back(-1);
        int pathC = 0, p = -1;
        size_t idx = trail_.size();
        std::vector<int> toclear;
        do {
            Clause& c = clauses_[confl];
            if (c.learnt) bump_clause(c);
            for (size_t k = (p < 0 ? 0 : 1); k < c.lits.size(); ++k) {
                const int q = c.lits[k], v = q >> 1;
                if (seen_[v] || level_[v] == 0) continue;
                seen_[v] = 1;
                toclear.push_back(v);
                bump_var(v);
                if (level_[v] >= level()) ++pathC;
                else out.push_back(q);
            }
            while (!seen_[trail_[--idx] >> 1]) {}
            p = trail_[idx];
            confl = reason_[p >> 1];
            seen_[p >> 1] = 0;
            --pathC;
        } while (pathC > 0);
        out[0] = p ^ 1;
        // local minimisation: drop literals implied by other literals of the clause
        size_t j = 1;
        for (size_t i = 1; i < out.size(); ++i) {
            const int v = out[i] >> 1, r = reason_[v];
            bool redundant = r >= 0;
            if (redundant) {
                const Clause& c = clauses_[r];
                for (size_t k = 1; k < c.lits.size(); ++k) {
                    const int u = c.lits[k] >> 1;
                    if (!seen_[u] && level_[u] > 0) { redundant = false; break; }
                }
            }
            if (!redundant) out[j++] = out[i];
        }
        out.resize(j);
        bt_level = 0;
        if (out.size() > 1) {
            size_t mi = 1;
            for (size_t i = 2; i < out.size(); ++i)
                if (level_[out[i] >> 1] > level_[out[mi] >> 1]) mi = i;
            std::swap(out[1], out[mi]);
            bt_level = level_[out[1] >> 1];
        }
        for (int v : toclear) seen_[v] = 0;
    }

    void backtrack(int lvl) {
        if (level() <= lvl) return;
        for (size_t i = trail_.size(); i > (size_t)trail_lim_[lvl]; --i) {
            const int v = trail_[i - 1] >> 1;
            phase_[v] = val_[v];
            val_[v] = -1;
            reason_[v] = -1;
            heap_insert(v);
        }
        trail_.resize(trail_lim_[lvl]);
        trail_lim_.resize(lvl);
        qhead_ = trail_.size();
    }

    void reduce_db() {
        std::vector<int> cand;
        for (int i : learnt_idx_) {
            Clause& c = clauses_[i];
            if (c.dead || c.lits.size() <= 2) continue;
            const int v = c.lits[0] >> 1;
            if (reason_[v] == i && value(c.lits[0]) == 1) continue;   // locked
            cand.push_back(i);
        }
        std::sort(cand.begin(), cand.end(), [&](int a, int b) { return clauses_[a].act < clauses_[b].act; });
        for (size_t i = 0; i < cand.size() / 2; ++i) {
            Clause& c = clauses_[cand[i]];
            c.dead = true;
            std::vector<int>().swap(c.lits);
        }
        std::vector<int> keep;
        for (int i : learnt_idx_)
            if (!clauses_[i].dead) keep.push_back(i);
        learnt_idx_.swap(keep);
    }

    int search(int64_t budget, int64_t conflict_limit, const std::atomic<int>* stop,
               std::chrono::steady_clock::time_point deadline) {
        std::vector<int> learnt;
        int64_t nconf = 0;
        for (;;) {
            const int confl = propagate();
            if (confl >= 0) {
                ++conflicts;
                ++nconf;
                if (level() == 0) return kUnsat;
                int bt;
                analyze(confl, learnt, bt);
                backtrack(bt);
                if (learnt.size() == 1) {
                    enqueue(learnt[0], -1);
                } else {
                    const int ci = add(learnt, true);
                    attach(ci);
                    learnt_idx_.push_back(ci);
                    bump_clause(clauses_[ci]);
                    enqueue(learnt[0], ci);
                }
                var_inc_ /= 0.95;
                cla_inc_ /= 0.999;
                if ((conflicts & 255) == 0) {
                    if (stop && stop->load(std::memory_order_relaxed)) { stopped_ = true; return kUnknown; }
                    if (std::chrono::steady_clock::now() > deadline) { stopped_ = true; return kUnknown; }
                }
                if (conflict_limit > 0 && conflicts >= conflict_limit) { stopped_ = true; return kUnknown; }
                continue;
            }
            if (nconf >= budget) {                               // restart (keeps assumptions re-applied)
                backtrack(0);
                return kUnknown;
            }
            if ((double)learnt_idx_.size() - (double)trail_.size() >= max_learnts_) reduce_db();
            int next_lit = -1;
            while (level() < (int)assumptions_.size()) {
                const int a = assumptions_[level()];
                const int x = value(a);
                if (x == 1) {
                    trail_lim_.push_back((int)trail_.size());         // already true: empty decision level
                } else if (x == 0) {
                    return kUnsatAssump;
                } else {
                    next_lit = a;
                    break;
                }
            }
            if (next_lit < 0) {
                int v = -1;
                while (!heap_.empty()) {
                    const int u = heap_pop();
                    if (val_[u] < 0) { v = u; break; }
                }
                if (v < 0) return kSat;
                next_lit = 2 * v + (phase_[v] == 1 ? 0 : 1);
                ++decisions;
            }
            trail_lim_.push_back((int)trail_.size());
            enqueue(next_lit, -1);
        }
    }
};

int to_internal(int32_t dimacs) { return 2 * (std::abs(dimacs) - 1) + (dimacs < 0 ? 1 : 0); }

bool build(Solver& s, int32_t V, int64_t C, const int64_t* ptr, const int32_t* lits) {
    std::vector<int> c;
    for (int64_t i = 0; i < C; ++i) {
        c.clear();
        for (int64_t j = ptr[i]; j < ptr[i + 1]; ++j) c.push_back(to_internal(lits[j]));
        if (!s.add_clause(c)) return false;
    }
    (void)V;
    return true;
}

bool check_args(int32_t V, int64_t C, const int64_t* ptr, const int32_t* lits) {
    if (V < 0 || C < 0 || (C > 0 && (!ptr || !lits))) return false;
    if (C > 0 && ptr[0] != 0) return false;
    for (int64_t i = 0; i < C; ++i)
        if (ptr[i + 1] < ptr[i]) return false;
    for (int64_t j = 0; C > 0 && j < ptr[C]; ++j)
        if (lits[j] == 0 || std::abs(lits[j]) > V) return false;
    return true;
}

}  // namespace cdcl
}  // namespace tsat

using namespace tsat::cdcl;

extern "C" tsat_status tsat_cdcl_solve(int32_t V, int64_t C, const int64_t* clause_ptr, const int32_t* dimacs_lits,
                                       int32_t n_assumptions, const int32_t* assumptions, int64_t conflict_limit,
                                       uint64_t seed, uint8_t* model_out, tsat_cdcl_result* out) {
    if (!out || !check_args(V, C, clause_ptr, dimacs_lits) || n_assumptions < 0 || (n_assumptions && !assumptions))
        return TSAT_E_ARG;
    for (int32_t i = 0; i < n_assumptions; ++i)
        if (assumptions[i] == 0 || std::abs(assumptions[i]) > V) return TSAT_E_ARG;
    try {
        const auto t0 = std::chrono::steady_clock::now();
        Solver s(V, seed);
        int r = build(s, V, C, clause_ptr, dimacs_lits) ? kUnknown : kUnsat;
        if (r != kUnsat) {
            std::vector<int> as;
            for (int32_t i = 0; i < n_assumptions; ++i) as.push_back(to_internal(assumptions[i]));
            r = s.solve(as, conflict_limit, nullptr, t0 + std::chrono::hours(24 * 365));
        }
        std::memset(out, 0, sizeof(*out));
        out->status = r;
        out->winner = -1;
        out->seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
        out->conflicts = s.conflicts;
        out->decisions = s.decisions;
        out->propagations = s.propagations;
        if (r == kSat && model_out)
            for (int32_t v = 0; v < V; ++v) model_out[v] = (uint8_t)(s.values()[v] == 1);
        return TSAT_OK;
    } catch (const std::bad_alloc&) {
        return TSAT_E_OOM;
    } catch (...) {
        return TSAT_E_ARG;
    }
}

extern "C" tsat_status tsat_cdcl_portfolio(int32_t V, int64_t C, const int64_t* clause_ptr, const int32_t* dimacs_lits,
                                           int32_t M, int32_t k, const int32_t* seeds, int32_t threads,
                                           int32_t unseeded, double time_limit_s, uint8_t* model_out,
                                           tsat_cdcl_result* out) {
    if (!out || !check_args(V, C, clause_ptr, dimacs_lits) || M < 0 || k < 0 || (M && k && !seeds) || threads < 1 ||
        !(time_limit_s > 0))
        return TSAT_E_ARG;
    for (int64_t i = 0; i < (int64_t)M * k; ++i)
        if (std::abs(seeds[i]) > V) return TSAT_E_ARG;
    try {
        const auto t0 = std::chrono::steady_clock::now();
        const auto deadline = t0 + std::chrono::microseconds((int64_t)(time_limit_s * 1e6));
        // jobs: the seeds in export order (best candidates first, l.286), then
        // the unseeded instance; with unseeded >= 1 it runs first on its own thread
        std::vector<int> jobs;
        if (unseeded) jobs.push_back(-1);
        for (int m = 0; m < M; ++m) jobs.push_back(m);
        std::atomic<int> next{0}, stop{0}, failed{0};
        std::mutex mu;
        tsat_cdcl_result best{};
        best.status = kUnknown;
        best.winner = -2;
        std::vector<uint8_t> model((size_t)V, 0);
        std::atomic<int> oom{0};
        auto work = [&](int tid) {
          try {                                 // no exception may leave a std::thread (terminate)
            for (;;) {
                const int j = next.fetch_add(1);
                if (j >= (int)jobs.size() || stop.load()) return;
                const int m = jobs[j];
                Solver s(V, (uint64_t)(m + 2) * 7919ull + (uint64_t)tid);
                int r = build(s, V, C, clause_ptr, dimacs_lits) ? kUnknown : kUnsat;
                if (r != kUnsat) {
                    std::vector<int> as;
                    if (m >= 0)
                        for (int i = 0; i < k; ++i) {
                            const int32_t x = seeds[(size_t)m * k + i];
                            if (x) as.push_back(to_internal(x));
                        }
                    r = s.solve(as, 0, &stop, deadline);
                }
                if (r == kUnsatAssump) { failed.fetch_add(1); continue; }
                if (r == kUnknown) continue;
                std::lock_guard<std::mutex> g(mu);
                if (best.status == kUnknown) {
                    best.status = r;                  // kSat, or kUnsat (the instance itself)
                    best.winner = m;
                    best.conflicts = s.conflicts;
                    best.decisions = s.decisions;
                    best.propagations = s.propagations;
                    if (r == kSat)
                        for (int32_t v = 0; v < V; ++v) model[v] = (uint8_t)(s.values()[v] == 1);
                    best.seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
                }
                stop.store(1);
                return;
            }
          } catch (...) {
            oom.store(1);
            stop.store(1);
          }
        };
        std::vector<std::thread> th;
        const int nt = std::max(1, std::min<int>(threads, (int)jobs.size()));
        for (int i = 0; i < nt; ++i) th.emplace_back(work, i);
        for (auto& x : th) x.join();
        if (oom.load()) return TSAT_E_OOM;
        *out = best;
        out->failed_seeds = failed.load();
        out->threads = nt;
        if (best.status == kUnknown) {
            out->winner = -2;
            out->seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
        }
        if (best.status == kSat && model_out) std::memcpy(model_out, model.data(), (size_t)V);
        return TSAT_OK;
    } catch (const std::bad_alloc&) {
        return TSAT_E_OOM;
    } catch (...) {
        return TSAT_E_ARG;
    }
}
