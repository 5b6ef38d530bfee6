// Host-side model IR for the B200 executor: the module tree, static SSA graphs,
// parameters and shard maps that Slapo's schedule primitives rewrite.
//
// Mirrors the reference's IR contract (same six node kinds, same attribute
// variant, same out-major Linear weight, same shard bookkeeping) so that a
// model scheduled with the reference API round-trips through slapo-model-v1
// JSON into this executor unchanged:
//   attrs / Error           proj/include/slapo/attrs.hpp:16-24
//   TensorSpec / ValueSpec  proj/include/slapo/tensor.hpp:22-103
//   graph (6 node kinds)    proj/include/slapo/graph.hpp:13-50
//   ParamDef / ShardInfo    proj/include/slapo/module.hpp:24-68
//   ModuleDef               proj/include/slapo/module.hpp:88-124
#pragma once

#include <cstdint>
#include <map>
#include <memory>
#include <optional>
#include <stdexcept>
#include <string>
#include <variant>
#include <vector>

namespace sb {

using i64 = std::int64_t;
using u64 = std::uint64_t;

using Attr = std::variant<i64, double, std::string, std::vector<i64>>;
using Attrs = std::map<std::string, Attr>;

struct Error : std::runtime_error {
    explicit Error(const std::string& m) : std::runtime_error(m) {}
};

// R1 sync-needs-shard, R2 distributed-needs-world, R3 needs-trace,
// R4 interface mismatch, R5 divisibility (proj/include/slapo/schedule.hpp:27-35).
struct RuleError : Error {
    RuleError(std::string r, const std::string& m) : Error(r + ": " + m), rule(std::move(r)) {}
    std::string rule;
};

std::optional<i64> get_int(const Attrs& a, const std::string& k);
std::optional<double> get_double(const Attrs& a, const std::string& k);
std::optional<std::string> get_str(const Attrs& a, const std::string& k);
std::optional<std::vector<i64>> get_ints(const Attrs& a, const std::string& k);
inline bool get_flag(const Attrs& a, const std::string& k) { return get_int(a, k).value_or(0) != 0; }

enum class Dtype { F32, F64 };
Dtype dtype_from(const std::string& s);
inline const char* dtype_str(Dtype d) { return d == Dtype::F32 ? "f32" : "f64"; }
inline int dtype_bytes(Dtype d) { return d == Dtype::F32 ? 4 : 8; }

struct TensorSpec {
    std::vector<i64> shape;
    Dtype dtype = Dtype::F64;
    i64 numel() const {
        i64 n = 1;
        for (i64 d : shape) n *= d;
        return n;
    }
    int rank() const { return (int)shape.size(); }
    bool operator==(const TensorSpec& o) const { return shape == o.shape && dtype == o.dtype; }
    bool operator!=(const TensorSpec& o) const { return !(*this == o); }
    std::string str() const;
};

struct ValueSpec {
    std::vector<TensorSpec> parts;
    bool tuple = false;
    ValueSpec() = default;
    explicit ValueSpec(TensorSpec t) : parts{std::move(t)} {}
    static ValueSpec of_tuple(std::vector<TensorSpec> p) {
        ValueSpec v;
        v.parts = std::move(p);
        v.tuple = true;
        return v;
    }
    const TensorSpec& one() const {
        if (tuple || parts.size() != 1) throw Error("value is not a single tensor");
        return parts[0];
    }
    bool operator==(const ValueSpec& o) const { return tuple == o.tuple && parts == o.parts; }
    std::string str() const;
};

// Host tensor (row-major, double payload), the reference's TensorValue.
struct HostTensor {
    TensorSpec spec;
    std::vector<double> data;
    HostTensor() = default;
    explicit HostTensor(TensorSpec s) : spec(std::move(s)), data((size_t)spec.numel(), 0.0) {}
    void round_f32() {
        if (spec.dtype == Dtype::F32)
            for (auto& x : data) x = (double)(float)x;
    }
};

// --------------------------------------------------------------------- graph
enum class NK { Input, ParamRef, CallModule, CallOp, GetItem, Output };
const char* nk_str(NK k);
NK nk_from(const std::string& s);

struct Node {
    int id = -1;
    NK kind = NK::Input;
    std::string op;      // call_op
    std::string target;  // call_module / param_ref
    std::vector<int> args;
    Attrs attrs;
};

struct Graph {
    std::vector<Node> nodes;
    std::vector<int> inputs;
    int out = -1;

    int pos(int id) const;
    const Node& at(int id) const;
    Node& at(int id);
    int max_id() const;
    const Node& out_node() const { return at(out); }
    void validate() const;
    Graph renumbered() const;
};
bool graphs_iso(const Graph& a, const Graph& b);

// Small builder with sequential ids.
struct GB {
    Graph g;
    int next = 0;
    int add(NK k, std::string op, std::string tgt, std::vector<int> args, Attrs at = {}) {
        Node n;
        n.id = next++;
        n.kind = k;
        n.op = std::move(op);
        n.target = std::move(tgt);
        n.args = std::move(args);
        n.attrs = std::move(at);
        if (k == NK::Input) g.inputs.push_back(n.id);
        g.nodes.push_back(std::move(n));
        return next - 1;
    }
    int input(Attrs a = {}) { return add(NK::Input, "", "", {}, std::move(a)); }
    int param(const std::string& p) { return add(NK::ParamRef, "", p, {}); }
    int call(const std::string& m, std::vector<int> a) { return add(NK::CallModule, "", m, std::move(a)); }
    int op(const std::string& o, std::vector<int> a, Attrs at = {}) { return add(NK::CallOp, o, "", std::move(a), std::move(at)); }
    int item(int src, i64 idx) { return add(NK::GetItem, "", "", {src}, Attrs{{"index", idx}}); }
    Graph finish(std::vector<int> results) {
        add(NK::Output, "", "", std::move(results));
        g.out = next - 1;
        g.validate();
        return std::move(g);
    }
};

// ------------------------------------------------------------------- modules
enum class Init { Normal, Uniform, Zeros, Ones };
const char* init_str(Init i);
Init init_from(const std::string& s);

struct ShardInfo {
    int axis = 0;
    int world = 1;
    int blocks = 1;
    std::vector<i64> full_shape;
    bool operator==(const ShardInfo& o) const {
        return axis == o.axis && world == o.world && blocks == o.blocks && full_shape == o.full_shape;
    }
};

struct Param {
    std::string name;
    TensorSpec spec;  // worker-local shape when sharded
    Init init = Init::Normal;
    u64 seed = 0;
    std::vector<u64> block_seeds;
    std::vector<double> values;
    std::optional<ShardInfo> shard;
    std::vector<i64> full_shape() const { return shard ? shard->full_shape : spec.shape; }
};

struct Module;
struct Child {
    std::string name;
    std::unique_ptr<Module> mod;
    Child(std::string n, Module m);
    Child(const Child& o);
    Child(Child&&) noexcept = default;
    Child& operator=(const Child& o);
    Child& operator=(Child&&) noexcept = default;
    ~Child();
};

struct Module {
    std::string name;
    std::string kind = "composite";
    std::vector<Param> params;
    std::vector<Child> children;
    std::optional<Graph> forward;
    Attrs attrs;

    bool composite() const { return kind == "composite"; }
    const Module* child(const std::string& seg) const;
    Module* child(const std::string& seg);
    const Module* resolve(const std::string& path) const;
    Module* resolve(const std::string& path);
    const Param* param(const std::string& n) const;
    Param* param(const std::string& n);
    const Param* resolve_param(const std::string& dotted) const;
    void add_child(const std::string& seg, Module m);
    void replace_child(const std::string& seg, Module m);
    void validate() const;
};

bool is_builtin_kind(const std::string& k);
bool modules_equal(const Module& a, const Module& b);

// paths: dot separated, `*` one segment, `**` any run
std::vector<std::string> split_path(const std::string& p);
std::string join(const std::string& a, const std::string& b);
std::string parent_of(const std::string& p);
std::string last_of(const std::string& p);
bool glob_match(const std::string& pattern, const std::string& concrete);
bool has_glob(const std::string& p);
std::vector<std::string> all_module_paths(const Module& root);
std::vector<std::string> expand_glob(const Module& root, const std::string& pattern);

// builtin constructors (proj/src/module.cpp:304-368)
Module make_linear(i64 in, i64 out, bool bias, u64 seed);
Module make_layernorm(i64 n, double eps, u64 seed);
Module make_dropout(double p, u64 seed);
Module make_embedding(i64 rows, i64 dim, u64 seed);

// parameter materialisation and shard index maps (proj/src/module.cpp:379-498)
HostTensor param_full(const Param& p);
HostTensor param_rank(const Param& p, int rank);
HostTensor slice_axis(const HostTensor& full, int axis, int world, int rank);
// Index map used by param_rank: local flat index -> full flat index.
void shard_index_map(const Param& p, int rank, std::vector<i64>& out);

// shape inference (proj/src/shape_inference.cpp)
bool is_builtin_op(const std::string& op);
ValueSpec infer_op(const std::string& op, const std::vector<const ValueSpec*>& args, const Attrs& a, int node_id);
int module_arity(const Module& m);
ValueSpec module_out_spec(const Module& m, const std::vector<TensorSpec>& ins);
std::map<int, ValueSpec> infer_graph(const Graph& g, const std::vector<TensorSpec>& ins, const Module& ctx);
std::vector<TensorSpec> declared_inputs(const Graph& g);
std::vector<TensorSpec> module_input_specs_at(const Module& root, const std::string& path);

// inputs (proj/src/executor.cpp:14-25)
HostTensor random_tensor(const TensorSpec& spec, u64 seed, u64 stream);
i64 embedding_row(double raw, i64 rows);

}  // namespace sb
