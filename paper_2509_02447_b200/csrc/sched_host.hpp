// Host planners of the CUDA-stream executor: the paper's Algorithm 1
// (adaptive stream allocation, reference sched.cpp:50-114) and Algorithm 2
// (resource-aware LPT mini-batch scheduling, sched.cpp:161-235), plus the
// warm-up statistics helper (sim.cpp:214-238). Plain C++; the device side only
// consumes the resulting plan.
#pragma once

#include <cstdint>
#include <functional>
#include <string>
#include <vector>

namespace qrm::sched {

struct Profile {
    double b0 = 1.0;
    std::vector<double> time;    // t[k] at baseline batch b0
    std::vector<double> memory;  // u[k] per sample
    // Optional GPU-aware extension (not in the reference): sat[k] = the largest
    // speedup concurrent streams give stage k (measured: a PCIe-bound transfer
    // stays near 1). Empty: the reference model, s streams = s times faster.
    std::vector<double> sat;
};

struct Plan {
    std::vector<int> streams;
    std::vector<int> minibatch;
    double bottleneck = 0.0;
};

struct Task {
    int id = 0;
    int tile_size = 0;
    double latency = 0.0;
    double memory = 0.0;
    int units = 1;
    int mb = 0;
};

struct Schedule {
    std::vector<std::vector<Task>> streams;
    std::vector<double> loads;
    int m_unit = 1;
};

// Error codes follow qrm_status: 0 ok, 1 invalid input, 3 infeasible.
double stage_time(const Profile& p, int k, int s, int m);
bool mem_ok(const std::vector<int>& s, const std::vector<int>& m, const std::vector<double>& u, double cap);
int allocate_streams(const Profile& p, int global_batch, int stream_budget, double m_cap, double epsilon,
                     int stall_cap, Plan& out, std::string& err);
int lpt_schedule(std::vector<Task> tasks, int stream_count, double lambda, double m_cap, int b_min,
                 int global_batch, Schedule& out, std::string& err);

// Median of `iters` timed runs per stage (ms), the clock injectable.
std::vector<double> measure_stages(const std::vector<std::function<void()>>& stages, int iters,
                                   const std::function<int64_t()>& now_ns);

}  // namespace qrm::sched
