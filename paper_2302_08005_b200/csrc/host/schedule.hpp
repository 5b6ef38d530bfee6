// The schedule language kept as the drop-in boundary: create_schedule and the
// primitives replace / shard / sync / checkpoint / trace / find / fuse /
// pipeline_split, replayed on a pristine copy by apply().
// Reference API: proj/include/slapo/schedule.hpp:37-109 (same names, argument
// meaning, rule errors R1-R5 and error texts), tracer.hpp, pattern.hpp,
// library.hpp.
#pragma once

#include <map>
#include <memory>

#include "ir.hpp"

namespace sb {

// ---------------------------------------------------------------- tracer
struct TraceSpec {
    std::vector<std::string> leaves;
    bool flatten = false;
};
Graph inline_call(const Graph& g, int call_node, const Graph& callee, const std::string& prefix);
int flatten_module(Module& target, const TraceSpec& spec, std::vector<std::string>* warnings);
void check_param_aliasing(const Module& root, const std::string& owner);

// --------------------------------------------------------------- pattern
struct Match {
    std::string site;
    std::vector<int> nodes;        // ascending graph ids
    std::map<int, int> binding;    // pattern core id -> graph id
};
std::vector<Match> find_matches(const Graph& g, const Graph& pattern, const Module* host);
std::vector<Match> find_module_calls(const Graph& g, const std::string& glob);
std::vector<int> escaping_values(const Graph& g, const std::vector<int>& nodes);
void validate_pattern(const Graph& p);

// --------------------------------------------------------------- library
Module make_attention_core(i64 head_dim, double p, u64 seed, bool causal = false);
Module make_qkv_composite(i64 hidden, u64 seed);
Module build_fused_qkv(const Module& old_qkv);
bool has_library_module(const std::string& n);
Module build_library_module(const std::string& n, const Module& old);
Module attention_reference_graph(const Module& ea);  // EfficientAttention semantics

// -------------------------------------------------------------- schedule
struct WorldConfig {
    int world_size = 1;
};

enum class Prim { Replace, Shard, Sync, Checkpoint, Trace, Find, Fuse, PipelineSplit };
const char* prim_str(Prim p);

struct Record {
    Prim prim = Prim::Trace;
    std::string site, library, pattern;
    std::vector<std::string> params;
    int axis = 0;
    std::string sync_type;
    TraceSpec trace;
    std::string after_child;
    std::string backend;
};

struct SplitAnnotation {
    std::string site, after_child;
};

struct ApplyResult {
    Module model;
    std::vector<SplitAnnotation> pipeline_splits;  // materialised by build_stage_plan (stages.hpp)
};

struct ScheduleState;

class Schedule {
public:
    Schedule(Module model, WorldConfig world);
    Schedule at(const std::string& path) const;
    const std::string& path() const { return path_; }
    std::vector<std::string> children() const;
    const Module& module() const;
    const Module& original() const;
    const WorldConfig& world() const;

    void trace(TraceSpec spec = {});
    void replace_with(const std::string& lib);
    void replace_at(const std::string& lib, const std::string& pattern);
    void shard(const std::vector<std::string>& params, int axis);
    void sync(const std::string& type);
    void checkpoint();
    void checkpoint_at(const std::string& pattern);
    std::vector<Match> find(const std::string& glob);
    std::vector<Match> find(const Graph& pattern);
    void fuse_at(const std::string& pattern, const std::string& backend = "composed");
    void pipeline_split(const std::string& after_child);
    void define_pattern(const std::string& name, Graph pattern);

    const std::vector<Record>& log() const;
    const std::vector<std::string>& warnings() const;
    ApplyResult apply() const;

    void set_deferred(bool d);
    void record_raw(Record r);

private:
    Schedule(std::shared_ptr<ScheduleState> s, std::string p) : st_(std::move(s)), path_(std::move(p)) {}
    void record(Record r);
    std::shared_ptr<ScheduleState> st_;
    std::string path_;
};

void check_record_rules(const Record& r, const std::vector<Record>& prior, const WorldConfig& w);
void apply_record(Module& model, const Record& r, const WorldConfig& w, const std::map<std::string, Graph>& patterns,
                  std::vector<std::string>* warnings);

// Line-oriented schedule scripts (proj/src/script.cpp:74-236 syntax).
void load_schedule_script(Schedule& s, const std::string& text);

// slapo-model-v1 JSON (proj/src/model_io.cpp)
Module load_model_json(const std::string& text);
std::string save_model_json(const Module& m);
Graph parse_graph_json(const std::string& text);

// Fixture models with the reference's seeds (proj/tests/support/fixtures.cpp).
struct BertConfig {
    int layers = 24;
    i64 hidden = 8, heads = 2, vocab = 28, batch = 4, seq = 4;
    double dropout_p = 0.1;
};
Module toy_bert(const BertConfig& c);
// f2: a GPT-Neo-style pre-LN decoder (causal attention) in the
// reference's module vocabulary, runnable by the oracle extension (oracle/causal_ext.py)
struct DecoderConfig {
    int layers = 2;
    i64 hidden = 8, heads = 2, vocab = 28, batch = 4, seq = 4;
    double dropout_p = 0.1;
};
Module gpt_neo(const DecoderConfig& c);
// f2: a T5-style encoder-decoder with cross-attention (BASELINE.json configs[4])
struct T5Config {
    int enc_layers = 2, dec_layers = 2;
    i64 hidden = 8, heads = 2, vocab = 28, batch = 4, enc_seq = 4, dec_seq = 4;
    double dropout_p = 0.1;
    bool tie_embeddings = true;  // one table for both id inputs (T5); false: enc_embed / dec_embed
};
Module t5(const T5Config& c);
Module tp_two_linear(i64 hidden, i64 inner, i64 batch);
Module fig3c_exact();
Module ffn_stack(int n, i64 hidden, i64 batch);
void convert_to_f32(Module& m);

}  // namespace sb
