// Reference-side drop-in binding: slapo::B200Executor with the
// method set of slapo::Executor (proj/include/slapo/executor.hpp:37-63), compiled
// into a program that uses the reference's headers and linked against
// libslapo_b200.so. It serialises the post-apply ModuleDef with the reference's
// own save_model (proj/include/slapo/model_io.hpp:20) and drives the C ABI of
// include/slapo_b200.h. tests/test_integration.py compiles it against
// /root/reference/proj/include (CPU) and runs it next to slapo::Executor (GPU).
#pragma once

#include <slapo_b200.h>

#include <string>
#include <vector>

#include "slapo/executor.hpp"
#include "slapo/model_io.hpp"
#include "slapo/schedule.hpp"

namespace slapo {

class B200Executor {
public:
    B200Executor(const ModuleDef& root, ExecMode mode, std::uint64_t seed, int world = 1, bool bf16 = false)
        : world_(world) {
        const std::string json = save_model(root);
        check(sb_model_from_json(json.c_str(), &model_));
        check(sb_executor_create(model_, mode == ExecMode::Train, seed, world, bf16 ? 1 : 0, /*fused=*/1, &ex_));
    }
    ~B200Executor() {
        sb_executor_free(ex_);
        sb_model_free(model_);
    }
    B200Executor(const B200Executor&) = delete;
    B200Executor& operator=(const B200Executor&) = delete;

    void set_nan_guard(bool on) { check(sb_executor_set_nan_guard(ex_, on ? 1 : 0)); }

    std::vector<TensorValue> forward(const std::vector<TensorValue>& inputs) {
        std::vector<const double*> ptrs;
        for (const auto& t : inputs) ptrs.push_back(t.data.data());
        check(sb_executor_forward(ex_, ptrs.data(), static_cast<int>(ptrs.size())));
        return outputs_of_rank(0);
    }

    std::vector<TensorValue> outputs_of_rank(int rank) const {
        int n = 0;
        check(sb_executor_num_outputs(ex_, rank, &n));
        std::vector<TensorValue> out;
        for (int i = 0; i < n; ++i) {
            size_t cnt = 0;
            std::int64_t dims[16];
            int nd = 16;
            check(sb_executor_output(ex_, rank, i, nullptr, 0, &cnt, dims, &nd));
            TensorValue t(TensorSpec{std::vector<std::int64_t>(dims, dims + nd), Dtype::F64});
            check(sb_executor_output(ex_, rank, i, t.data.data(), t.data.size(), &cnt, dims, &nd));
            out.push_back(std::move(t));
        }
        return out;
    }

    GradientMap backward() { return backward_all_ranks()[0]; }

    std::vector<GradientMap> backward_all_ranks() {
        check(sb_executor_backward(ex_));
        std::vector<GradientMap> maps(static_cast<size_t>(world_));
        for (int r = 0; r < world_; ++r) {
            int n = 0;
            char name[4096];
            check(sb_executor_num_grads(ex_, r, &n));
            for (int i = 0; i < n; ++i) {
                check(sb_executor_grad_name(ex_, r, i, name, sizeof name));
                size_t cnt = 0;
                check(sb_executor_grad(ex_, r, name, nullptr, 0, &cnt));
                std::vector<double> v(cnt);
                check(sb_executor_grad(ex_, r, name, v.data(), cnt, &cnt));
                maps[static_cast<size_t>(r)].params[name] =
                    TensorValue(TensorSpec{{static_cast<std::int64_t>(cnt)}, Dtype::F64}, std::move(v));
            }
        }
        return maps;
    }

    std::int64_t collective_invocations() const {
        std::int64_t c = 0;
        check(sb_executor_collectives(ex_, &c));
        return c;
    }
    std::int64_t ledger_bytes() const {
        std::int64_t b = 0;
        check(sb_executor_ledger(ex_, &b));
        return b;
    }

private:
    static void check(int rc) {
        if (rc == 2) throw RuleError(std::string(sb_last_error()).substr(0, 2), sb_last_error());
        if (rc != 0) throw Error(sb_last_error());
    }
    int world_ = 1;
    sb_model* model_ = nullptr;
    sb_executor* ex_ = nullptr;
};

}  // namespace slapo
