// B200 executor: the drop-in replacement for slapo::Executor
// (proj/include/slapo/executor.hpp:37-63). Same method set — forward,
// outputs_of_rank, backward, backward_all_ranks, ledger, collective_invocations,
// set_nan_guard — but the post-apply module is lowered once to a static device
// plan per rank and every op runs as an sm_100a kernel.
//
// Two placements of the `world` ranks:
//   * Local: all ranks on the current device, collectives are device-side sums in
//     rank-ascending order (the reference's lockstep simulator, executor.cpp:812-839,
//     with the same semantics) — used for parity at world > 1 on one GPU;
//   * Nccl: this process is rank `rank` of `world` processes (one per GPU),
//     collectives go through NCCL over NVLink.
#pragma once

#include <map>
#include <memory>
#include <string>
#include <vector>

#include "plan.hpp"

namespace sb {

// the process's NCCL (dlopen handle; nullptr if none): executor.cpp
void* nccl_handle();

struct CommConfig {
    bool nccl = false;
    int rank = 0;                // nccl: this process's rank
    std::vector<char> unique_id;  // nccl: 128-byte ncclUniqueId from rank 0
};

struct GradMap {
    std::map<std::string, HostTensor> params;
    std::vector<HostTensor> inputs;
};

class ExecutorImpl;

// a device-resident tensor of an executor (contiguous)
struct DeviceTensor {
    void* ptr;
    DT dt;
    i64 numel;
    std::vector<i64> shape;
};

class Executor {
public:
    Executor(const Module& root, bool train, u64 seed, int world, DT compute, const CommConfig& comm = {},
             bool fused_kernels = true);
    ~Executor();

    void set_nan_guard(bool on);
    std::vector<HostTensor> forward(const std::vector<HostTensor>& inputs);
    std::vector<HostTensor> outputs_of_rank(int rank) const;
    GradMap backward();                  // rank 0 (or this process's rank)
    std::vector<GradMap> backward_all_ranks();
    i64 ledger_bytes() const;
    i64 collective_invocations() const;

    // ---- device-resident stepping (bench / e2e) ----
    void upload_inputs(const std::vector<HostTensor>& inputs);  // H2D (pageable)
    void upload_inputs_raw(const double* const* inputs, int n);  // sizes from the plan
    void forward_uploaded();                                      // forward on already-uploaded inputs
    void set_inputs_device(int idx, const void* dptr);          // copy from a device f64 buffer
    void run_forward();   // enqueue forward
    void run_backward();  // enqueue backward
    void enqueue_loss(float* dloss);  // loss = sum of outputs (device fp32 scalar)
    void capture_graph();             // capture run_forward+run_backward into a CUDA graph
    void launch_graph();
    void synchronize();
    void* stream() const;
    int kernel_launches_per_step() const;  // kernel nodes of the captured step graph
    float time_steps(int steps, bool use_graph);  // device ms of `steps` fwd+bwd, CUDA events on our stream
    float time_e2e(int steps, const double* const* inputs, int n, bool use_graph, float* last_loss);
    std::string describe() const;  // plan summary (ops, bytes)
    size_t device_bytes() const;
    void* input_device_ptr(int idx) const;
    // kernel-level timing of one op kind (bench roofline): returns the ms of
    // all launches of op kind `k` inside one forward+backward, measured with events.
    std::vector<std::pair<std::string, float>> profile_step();

    // ---- pipeline-stage hooks (f1, csrc/host/pipeline_exec.cpp) ----
    void set_accumulate_param_grads(bool on);  // parameter gradients += across backward calls
    void zero_param_grads();                   // (enqueued)
    void set_output_grad_seed(int idx, const void* dptr, DT dt);  // backward seeds output idx from dptr (nullptr: ones)
    DeviceTensor output_device(int idx) const;
    DeviceTensor input_grad_device(int idx) const;
    void set_input_from_device(int idx, const void* src, DT dt);  // (enqueued) cast into input idx
    std::vector<GradMap> grads_all_ranks();                        // download the current gradients
    // in-place sum over the executor's ranks on `stream` (NCCL executors; identity at world 1)
    void all_reduce_device(void* buf, i64 n, DT dt, void* stream);

private:
    std::unique_ptr<ExecutorImpl> impl_;
};

}  // namespace sb
