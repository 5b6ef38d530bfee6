// Pipeline-parallel training step over the stages of a pipeline_split plan
// (the reference's run_pipeline, proj/src/executor.cpp:1531-1579,
// extended to a training step).
//
// GPipe with re-materialisation: the batch is cut into M micro-batches along
// dim 0; every stage runs on its own device (a device list; stages may share a
// device) through its own Executor planned for one micro-batch. Forward: for each
// micro-batch the stages run in order, each stage's produced values are stashed
// on the consumer's device (peer copy over NVLink when the devices differ) — only
// stage-boundary values are kept per micro-batch. Backward: micro-batches in
// reverse, stages in reverse; a stage first recomputes its forward from the
// stashed inputs (GPipe's re-materialisation), then runs its backward seeded with
// the gradient of its produced values (ones for model outputs, the loss being the
// sum of the outputs as in Executor::backward, plus the input gradients of every
// consumer stage, summed), accumulating parameter gradients across micro-batches.
// All of it is enqueued on the stages' streams with events between them: stages
// on different devices overlap across micro-batches.
//
// Semantics per micro-batch are those of run_pipeline: each stage executes its
// module with the executor seed on micro-batch-shaped tensors, so dropout draws
// use micro-batch-local indices (every micro-batch of a stage sees the same
// masks, exactly as the reference's run_forward per chunk does).
#pragma once

#include <memory>
#include <string>
#include <vector>

#include "executor.hpp"
#include "stages.hpp"

namespace sb {

// One process per (stage, tensor-parallel rank): rank = stage * tp + tp_rank of `world` =
// stages * tp processes. Stage-boundary values move with ncclSend / ncclRecv on a
// pipeline communicator (pp_uid) between ranks of equal tp_rank; the stage's own
// tensor parallelism runs on an NCCL communicator of its tp ranks (tp_uid, one per stage).
struct PipeDist {
    int rank = -1, world = 0;
    std::vector<char> pp_uid, tp_uid;
};

// The per-rank transfer program of a distributed pipeline step (pure function of the plan):
// forward, micro-batch m ascending: receive the remote inputs (sorted by producer stage,
// output index), run, send each output to each remote consumer (stage order); backward,
// m descending: receive the consumers' input gradients of each output (output index,
// consumer stage order), run, send the remote inputs' gradients to their producers (sorted
// as the forward receives). A pair of ranks thus posts matching transfers in the same
// order in both directions; tests/test_pipeline_program_cpu.py checks matching and
// deadlock freedom under rendezvous semantics over gloo and in simulation.
struct PipeStep {
    enum Kind : int { FwdRecv = 0, FwdRun = 1, FwdSend = 2, BwdRecv = 3, BwdRun = 4, BwdSend = 5 };
    Kind kind;
    int m, idx, peer;  // idx: the stage's input (Recv / BwdSend) or output (Send / BwdRecv) index
    std::string value;
};
std::vector<PipeStep> pipe_program(const StagePlan& plan, int micro, int tp, int rank);

class PipelineExecutor {
public:
    // tp > 1: every stage runs its (sharded) module on tp lockstep ranks of its device
    // (tensor parallelism inside the stage; stage-boundary values are replicated)
    PipelineExecutor(const StagePlan& plan, int micro_batches, bool train, u64 seed, DT compute,
                     std::vector<int> devices = {}, bool fused_kernels = true, int tp = 1,
                     const PipeDist* dist = nullptr);
    ~PipelineExecutor();

    // GPipe forward of every micro-batch; the model outputs concatenated along dim 0
    std::vector<HostTensor> forward(const std::vector<HostTensor>& inputs);
    std::vector<HostTensor> forward_raw(const double* const* inputs, int n);  // full-batch f64 inputs
    // backward of sum(outputs) over all micro-batches (requires forward): per stage and
    // tensor-parallel rank (slot stage * tp + rank), its parameter gradients summed over
    // micro-batches (stage-local names) and the gradients of the model inputs it consumes
    // (concatenated over micro-batches)
    std::vector<GradMap> backward();
    int tp() const;
    // device ms of `steps` full training steps (forward + backward of every
    // micro-batch) on already-uploaded inputs (the last forward's); use_graph: the step is
    // captured once into a CUDA graph (stages on one device) and replayed
    float time_steps(int steps, bool use_graph = true);
    int num_stages() const;
    int micro_batches() const;

private:
    struct Impl;
    std::unique_ptr<Impl> impl_;
};

}  // namespace sb
