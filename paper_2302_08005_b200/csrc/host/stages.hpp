// Pipeline stages materialised from pipeline_split annotations (SURVEY.md
// §8(f) f1): the reference's PipelineStagePlan (proj/include/slapo/pipeline.hpp:14-40).
#pragma once

#include <string>
#include <vector>

#include "ir.hpp"
#include "schedule.hpp"

namespace sb {

struct Stage {
    Module module;
    std::vector<std::string> consumes;  // ordered, match the module's input nodes
    std::vector<std::string> produces;  // ordered, match the module's results
};

struct StagePlan {
    std::vector<Stage> stages;
    std::vector<std::string> model_inputs;   // names bound to the original model inputs
    std::vector<std::string> model_outputs;  // names of the original model results
};

// build_pipeline_plan (proj/src/pipeline.cpp:343-420). The input model is not modified.
StagePlan build_stage_plan(const Module& model, const std::vector<SplitAnnotation>& splits);

}  // namespace sb
