// Analytical step-time / memory model and checkpoint-ratio helper: the
// reference's cost model (proj/include/slapo/costmodel.hpp:12-59,
// proj/src/costmodel.cpp) over this library's IR, plus the B200 calibration
// of its constants (measured on this pool's B200s).
#pragma once

#include <cstdint>
#include <string>

#include "ir.hpp"

namespace sb {

struct CostConstants {  // costmodel.hpp:15-20 (configuration, not ground truth)
    double device_flops_per_s = 1e12;
    double link_bytes_per_s = 1e10;
    double kernel_launch_overhead_s = 1e-6;
    double optimizer_state_multiplier = 2.0;
};

struct CostReport {  // costmodel.hpp:22-35
    double step_time_s = 0.0;
    i64 flops = 0;
    i64 recompute_flops = 0;
    i64 launches = 0;
    i64 collective_bytes = 0;
    i64 param_bytes = 0;
    i64 activation_bytes = 0;
    i64 peak_memory_bytes = 0;
    bool oom = false;
    double throughput_samples_per_s = 0.0;
    std::string to_text() const;
};

struct EstimateOptions {  // costmodel.hpp:37-43
    i64 batch = 0;
    int micro_batches = 1;
    int world_size = 1;
    i64 device_memory_bytes = 16LL * 1024 * 1024 * 1024;
    CostConstants constants;
};

CostReport estimate(const Module& model, const EstimateOptions& opts);
int apply_checkpoint_ratio(Module& model, const std::string& container, double ratio);

}  // namespace sb
