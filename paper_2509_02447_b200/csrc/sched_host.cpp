#include "sched_host.hpp"

#include <algorithm>
#include <cmath>
#include <numeric>

namespace qrm::sched {

double stage_time(const Profile& p, int k, int s, int m) {
    // TIME(k, s, m) = t[k] * (m / b0) / s (sched.cpp:27-30); with measured
    // saturation, the s streams' speedup is capped at sat[k].
    double par = static_cast<double>(s);
    if (!p.sat.empty()) par = std::min(par, std::max(1.0, p.sat[k]));
    return p.time[k] * (static_cast<double>(m) / p.b0) / par;
}

bool mem_ok(const std::vector<int>& s, const std::vector<int>& m, const std::vector<double>& u, double cap) {
    double used = 0.0;
    for (size_t k = 0; k < s.size(); ++k) used += static_cast<double>(s[k]) * static_cast<double>(m[k]) * u[k];
    return used <= cap;
}

static double worst_stage(const Profile& p, const std::vector<int>& s, const std::vector<int>& m) {
    double w = 0.0;
    for (size_t k = 0; k < s.size(); ++k) w = std::max(w, stage_time(p, static_cast<int>(k), s[k], m[k]));
    return w;
}

int allocate_streams(const Profile& p, int B, int P, double m_cap, double eps, int stall_cap, Plan& out,
                     std::string& err) {
    const int K = static_cast<int>(p.time.size());
    if (K == 0) return err = "profile has no stages", 1;
    if (p.memory.size() != p.time.size()) return err = "profile time/memory length mismatch", 1;
    if (p.b0 < 1.0) return err = "baseline batch must be >= 1", 1;
    for (double t : p.time)
        if (!(t > 0.0)) return err = "stage times must be positive", 1;
    for (double u : p.memory)
        if (u < 0.0) return err = "per-sample memory must be nonnegative", 1;
    if (P < K) return err = "stream budget below stage count", 1;
    if (!p.sat.empty() && p.sat.size() != p.time.size()) return err = "profile saturation length mismatch", 1;
    if (B < 1) return err = "global batch must be >= 1", 1;

    // (1) one stream per stage; the largest uniform mini-batch that fits M_cap,
    // at most the global batch. (The reference casts floor(M_cap / sum u) to
    // int, undefined above INT_MAX; here it is clamped to B, the documented
    // intent of sched.cpp:56-59.)
    std::vector<int> s(K, 1);
    const double per_unit = std::accumulate(p.memory.begin(), p.memory.end(), 0.0);
    long long uniform = B;
    if (per_unit > 0.0) {
        const double fit = std::floor(m_cap / per_unit);
        if (fit < static_cast<double>(uniform)) uniform = static_cast<long long>(fit);
    }
    if (uniform < 1) return err = "memory cap cannot fit one sample per stage", 3;
    std::vector<int> m(K, static_cast<int>(uniform));
    double bn = worst_stage(p, s, m);

    // (2) greedy: add the single stream with the largest bottleneck reduction
    // while the gain exceeds epsilon, within budget P and M_cap; stop after
    // stall_cap rounds without an accepted move.
    for (int stall = 0; stall < stall_cap;) {
        int best = -1;
        double gain = 0.0;
        const int used = std::accumulate(s.begin(), s.end(), 0);
        for (int k = 0; k < K; ++k) {
            ++s[k];
            if (used + 1 <= P && mem_ok(s, m, p.memory, m_cap)) {
                const double d = bn - worst_stage(p, s, m);
                if (d > gain) {
                    gain = d;
                    best = k;
                }
            }
            --s[k];
        }
        if (best >= 0 && gain > eps) {
            ++s[best];
            bn = worst_stage(p, s, m);
            stall = 0;
        } else {
            ++stall;
        }
    }

    // (3) one levelling pass: stages under half the bottleneck double their
    // mini-batch up to m_unit = max(1, B / sum s), if memory allows.
    const int total = std::accumulate(s.begin(), s.end(), 0);
    const int m_unit = std::max(1, B / total);
    for (int k = 0; k < K; ++k) {
        if (stage_time(p, k, s[k], m[k]) < bn / 2.0) {
            const int keep = m[k];
            m[k] = std::min(m_unit, 2 * m[k]);
            if (!mem_ok(s, m, p.memory, m_cap)) m[k] = keep;
        }
    }
    out.streams = s;
    out.minibatch = m;
    out.bottleneck = worst_stage(p, s, m);
    return 0;
}

int lpt_schedule(std::vector<Task> tasks, int S, double lambda, double m_cap, int b_min, int B, Schedule& out,
                 std::string& err) {
    if (S < 1) return err = "need at least one stream", 1;
    if (b_min < 1) return err = "minimum mini-batch must be >= 1", 1;
    for (const Task& t : tasks)
        if (!(t.latency > 0.0) || t.units < 1) return err = "tasks must have positive latency and units", 1;
    out.streams.assign(S, {});
    out.loads.assign(S, 0.0);
    // Pool ascending by (latency, -id): the back is the longest task, lowest id first on ties.
    auto before = [](const Task& a, const Task& b) { return a.latency != b.latency ? a.latency < b.latency : a.id > b.id; };
    std::sort(tasks.begin(), tasks.end(), before);
    double placed_mem = 0.0;
    int placed = 0;
    while (!tasks.empty()) {
        Task task = tasks.back();
        tasks.pop_back();
        const int target = static_cast<int>(std::min_element(out.loads.begin(), out.loads.end()) - out.loads.begin());
        const double least = out.loads[target];
        const bool balanced = std::isinf(lambda) || least + task.latency <= (1.0 + lambda) * least;
        if (balanced && placed_mem + task.memory <= m_cap) {
            out.streams[target].push_back(task);
            out.loads[target] += task.latency;
            placed_mem += task.memory;
            ++placed;
            continue;
        }
        // Shard b_min units off the task (latency/memory pro rata, remainder
        // keeps the exact complement) and return the rest to the pool.
        Task head = task;
        bool has_rest = false;
        Task rest;
        if (task.units > b_min) {
            const double frac = static_cast<double>(b_min) / task.units;
            head.units = b_min;
            head.latency = task.latency * frac;
            head.memory = task.memory * frac;
            rest = task;
            rest.units = task.units - b_min;
            rest.latency = task.latency - head.latency;
            rest.memory = task.memory - head.memory;
            has_rest = true;
        }
        if (placed_mem + head.memory > m_cap) return err = "memory cap violated even at minimum shard size", 3;
        out.streams[target].push_back(head);
        out.loads[target] += head.latency;
        placed_mem += head.memory;
        ++placed;
        if (has_rest) tasks.insert(std::lower_bound(tasks.begin(), tasks.end(), rest, before), rest);
    }
    out.m_unit = std::max(b_min, placed ? B / placed : b_min);
    for (auto& st : out.streams)
        for (Task& t : st) t.mb = out.m_unit;
    return 0;
}

std::vector<double> measure_stages(const std::vector<std::function<void()>>& stages, int iters,
                                   const std::function<int64_t()>& now_ns) {
    std::vector<double> med;
    for (const auto& run : stages) {
        std::vector<double> v;
        for (int i = 0; i < iters; ++i) {
            const int64_t a = now_ns();
            run();
            v.push_back(static_cast<double>(now_ns() - a) / 1e6);
        }
        std::sort(v.begin(), v.end());
        double x = v[v.size() / 2];
        if (v.size() % 2 == 0) x = 0.5 * (x + v[v.size() / 2 - 1]);
        med.push_back(std::max(x, 1e-6));
    }
    return med;
}

}  // namespace qrm::sched
