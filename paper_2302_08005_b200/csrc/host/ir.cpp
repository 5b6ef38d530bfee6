// IR core: attributes, graphs, module tree, paths, builtin constructors,
// parameter materialisation + shard index maps, shape inference.
// Reference contract: proj/src/{tensor,graph,module,shape_inference}.cpp.
#include "ir.hpp"

#include <algorithm>
#include <functional>
#include <set>
#include <sstream>
#include <thread>
#include <unordered_map>
#include <unordered_set>

#include "rng.hpp"

namespace sb {

// ------------------------------------------------------------------- attrs
std::optional<i64> get_int(const Attrs& a, const std::string& k) {
    auto it = a.find(k);
    if (it == a.end()) return std::nullopt;
    if (auto p = std::get_if<i64>(&it->second)) return *p;
    return std::nullopt;
}
std::optional<double> get_double(const Attrs& a, const std::string& k) {
    auto it = a.find(k);
    if (it == a.end()) return std::nullopt;
    if (auto p = std::get_if<double>(&it->second)) return *p;
    if (auto p = std::get_if<i64>(&it->second)) return (double)*p;
    return std::nullopt;
}
std::optional<std::string> get_str(const Attrs& a, const std::string& k) {
    auto it = a.find(k);
    if (it == a.end()) return std::nullopt;
    if (auto p = std::get_if<std::string>(&it->second)) return *p;
    return std::nullopt;
}
std::optional<std::vector<i64>> get_ints(const Attrs& a, const std::string& k) {
    auto it = a.find(k);
    if (it == a.end()) return std::nullopt;
    if (auto p = std::get_if<std::vector<i64>>(&it->second)) return *p;
    return std::nullopt;
}

Dtype dtype_from(const std::string& s) {
    if (s == "f32") return Dtype::F32;
    if (s == "f64") return Dtype::F64;
    throw Error("unknown dtype '" + s + "' (expected f32 or f64)");
}

std::string TensorSpec::str() const {
    std::ostringstream o;
    o << "(";
    for (size_t i = 0; i < shape.size(); ++i) o << (i ? "," : "") << shape[i];
    o << "):" << dtype_str(dtype);
    return o.str();
}
std::string ValueSpec::str() const {
    if (!tuple) return parts.empty() ? "()" : parts[0].str();
    std::string s = "tuple[";
    for (size_t i = 0; i < parts.size(); ++i) s += (i ? ", " : "") + parts[i].str();
    return s + "]";
}

// ------------------------------------------------------------------- graph
const char* nk_str(NK k) {
    switch (k) {
        case NK::Input: return "input";
        case NK::ParamRef: return "param_ref";
        case NK::CallModule: return "call_module";
        case NK::CallOp: return "call_op";
        case NK::GetItem: return "get_item";
        case NK::Output: return "output";
    }
    return "?";
}
NK nk_from(const std::string& s) {
    static const std::map<std::string, NK> m = {{"input", NK::Input},          {"param_ref", NK::ParamRef},
                                                {"call_module", NK::CallModule}, {"call_op", NK::CallOp},
                                                {"get_item", NK::GetItem},     {"output", NK::Output}};
    auto it = m.find(s);
    if (it == m.end()) throw Error("unknown node kind '" + s + "'");
    return it->second;
}

int Graph::pos(int id) const {
    for (size_t i = 0; i < nodes.size(); ++i)
        if (nodes[i].id == id) return (int)i;
    return -1;
}
const Node& Graph::at(int id) const {
    int p = pos(id);
    if (p < 0) throw Error("no node with id " + std::to_string(id));
    return nodes[p];
}
Node& Graph::at(int id) {
    int p = pos(id);
    if (p < 0) throw Error("no node with id " + std::to_string(id));
    return nodes[p];
}
int Graph::max_id() const {
    int m = -1;
    for (auto& n : nodes) m = std::max(m, n.id);
    return m;
}
void Graph::validate() const {
    std::unordered_set<int> seen;
    int nout = 0, nin = 0;
    for (auto& n : nodes) {
        if (seen.count(n.id)) throw Error("duplicate node id " + std::to_string(n.id));
        for (int a : n.args)
            if (!seen.count(a))
                throw Error("node " + std::to_string(n.id) + " references id " + std::to_string(a) +
                            " that does not precede it");
        seen.insert(n.id);
        nout += n.kind == NK::Output;
        nin += n.kind == NK::Input;
        if (n.kind == NK::GetItem) {
            if (n.args.size() != 1) throw Error("get_item expects exactly one arg");
            if (!get_int(n.attrs, "index")) throw Error("get_item node " + std::to_string(n.id) + " missing index attr");
        }
    }
    if (nout != 1) throw Error("graph must have exactly 1 output node, has " + std::to_string(nout));
    if (nin < 1) throw Error("graph must have at least 1 input node");
    if (out < 0 || nodes.back().id != out || nodes.back().kind != NK::Output)
        throw Error("output node must be last and match output_id");
    for (int i : inputs)
        if (!seen.count(i)) throw Error("input_ids entry not present in graph");
}
Graph Graph::renumbered() const {
    std::unordered_map<int, int> re;
    int k = 0;
    for (auto& n : nodes) re[n.id] = k++;
    Graph g;
    for (auto n : nodes) {
        n.id = re[n.id];
        for (auto& a : n.args) a = re[a];
        g.nodes.push_back(std::move(n));
    }
    for (int i : inputs) g.inputs.push_back(re[i]);
    g.out = re.at(out);
    return g;
}
bool graphs_iso(const Graph& a, const Graph& b) {
    Graph x = a.renumbered(), y = b.renumbered();
    if (x.nodes.size() != y.nodes.size() || x.inputs != y.inputs || x.out != y.out) return false;
    for (size_t i = 0; i < x.nodes.size(); ++i) {
        auto &p = x.nodes[i], &q = y.nodes[i];
        if (p.id != q.id || p.kind != q.kind || p.op != q.op || p.target != q.target || p.args != q.args ||
            p.attrs != q.attrs)
            return false;
    }
    return true;
}

// ----------------------------------------------------------------- modules
const char* init_str(Init i) {
    switch (i) {
        case Init::Normal: return "normal";
        case Init::Uniform: return "uniform";
        case Init::Zeros: return "zeros";
        case Init::Ones: return "ones";
    }
    return "?";
}
Init init_from(const std::string& s) {
    if (s == "normal") return Init::Normal;
    if (s == "uniform") return Init::Uniform;
    if (s == "zeros") return Init::Zeros;
    if (s == "ones") return Init::Ones;
    throw Error("unknown init scheme '" + s + "'");
}

Child::Child(std::string n, Module m) : name(std::move(n)), mod(std::make_unique<Module>(std::move(m))) {}
Child::Child(const Child& o) : name(o.name), mod(o.mod ? std::make_unique<Module>(*o.mod) : nullptr) {}
Child& Child::operator=(const Child& o) {
    if (this != &o) {
        name = o.name;
        mod = o.mod ? std::make_unique<Module>(*o.mod) : nullptr;
    }
    return *this;
}
Child::~Child() = default;

const Module* Module::child(const std::string& seg) const {
    for (auto& c : children)
        if (c.name == seg) return c.mod.get();
    return nullptr;
}
Module* Module::child(const std::string& seg) {
    for (auto& c : children)
        if (c.name == seg) return c.mod.get();
    return nullptr;
}
const Module* Module::resolve(const std::string& path) const {
    const Module* cur = this;
    if (path.empty()) return cur;
    for (auto& s : split_path(path)) {
        cur = cur->child(s);
        if (!cur) return nullptr;
    }
    return cur;
}
Module* Module::resolve(const std::string& path) {
    return const_cast<Module*>(static_cast<const Module*>(this)->resolve(path));
}
const Param* Module::param(const std::string& n) const {
    for (auto& p : params)
        if (p.name == n) return &p;
    return nullptr;
}
Param* Module::param(const std::string& n) {
    for (auto& p : params)
        if (p.name == n) return &p;
    return nullptr;
}
const Param* Module::resolve_param(const std::string& dotted) const {
    auto d = dotted.rfind('.');
    if (d == std::string::npos) return param(dotted);
    const Module* o = resolve(dotted.substr(0, d));
    return o ? o->param(dotted.substr(d + 1)) : nullptr;
}
void Module::add_child(const std::string& seg, Module m) {
    if (child(seg)) throw Error("duplicate submodule name '" + seg + "' in module '" + name + "'");
    children.emplace_back(seg, std::move(m));
}
void Module::replace_child(const std::string& seg, Module m) {
    for (auto& c : children)
        if (c.name == seg) {
            *c.mod = std::move(m);
            return;
        }
    throw Error("unknown submodule '" + seg + "' in module '" + name + "'");
}
bool is_builtin_kind(const std::string& k) {
    static const std::set<std::string> s = {"Linear", "LayerNorm", "Dropout", "Embedding", "FusedQKV",
                                            "EfficientAttention"};
    return s.count(k) > 0;
}
void Module::validate() const {
    if (!composite() && !is_builtin_kind(kind)) throw Error("module '" + name + "' has unknown kind '" + kind + "'");
    std::set<std::string> cn, pn;
    for (auto& c : children) {
        if (c.name.empty() || c.name.find('.') != std::string::npos)
            throw Error("invalid submodule segment '" + c.name + "'");
        if (!cn.insert(c.name).second) throw Error("duplicate submodule name '" + c.name + "' in module '" + name + "'");
    }
    for (auto& p : params) {
        if (!pn.insert(p.name).second) throw Error("duplicate param name '" + p.name + "' in module '" + name + "'");
        for (i64 d : p.spec.shape)
            if (d < 1) throw Error("tensor dimension must be >= 1, got " + std::to_string(d));
    }
    if (composite()) {
        if (!forward) throw Error("composite module '" + name + "' missing forward graph");
        forward->validate();
        for (auto& n : forward->nodes) {
            if (n.kind == NK::CallModule && !resolve(n.target))
                throw Error("unknown submodule '" + n.target + "' referenced by module '" + name + "'");
            if (n.kind == NK::ParamRef && !resolve_param(n.target))
                throw Error("unknown param '" + n.target + "' referenced by module '" + name + "'");
        }
    }
    for (auto& c : children) c.mod->validate();
}
bool modules_equal(const Module& a, const Module& b) {
    if (a.kind != b.kind || a.attrs != b.attrs || a.params.size() != b.params.size()) return false;
    for (size_t i = 0; i < a.params.size(); ++i) {
        auto &p = a.params[i], &q = b.params[i];
        if (p.name != q.name || p.spec != q.spec || p.init != q.init || p.seed != q.seed ||
            p.block_seeds != q.block_seeds || p.values != q.values || p.shard.has_value() != q.shard.has_value())
            return false;
        if (p.shard && !(*p.shard == *q.shard)) return false;
    }
    if (a.forward.has_value() != b.forward.has_value()) return false;
    if (a.forward && !graphs_iso(*a.forward, *b.forward)) return false;
    if (a.children.size() != b.children.size()) return false;
    for (size_t i = 0; i < a.children.size(); ++i)
        if (a.children[i].name != b.children[i].name || !modules_equal(*a.children[i].mod, *b.children[i].mod))
            return false;
    return true;
}

// ------------------------------------------------------------------- paths
std::vector<std::string> split_path(const std::string& p) {
    std::vector<std::string> out;
    if (p.empty()) return out;
    size_t s = 0;
    while (true) {
        size_t d = p.find('.', s);
        std::string seg = p.substr(s, d == std::string::npos ? std::string::npos : d - s);
        if (seg.empty()) throw Error("empty segment in path '" + p + "'");
        out.push_back(seg);
        if (d == std::string::npos) break;
        s = d + 1;
    }
    return out;
}
std::string join(const std::string& a, const std::string& b) {
    if (a.empty()) return b;
    if (b.empty()) return a;
    return a + "." + b;
}
std::string parent_of(const std::string& p) {
    auto d = p.rfind('.');
    return d == std::string::npos ? std::string() : p.substr(0, d);
}
std::string last_of(const std::string& p) {
    auto d = p.rfind('.');
    return d == std::string::npos ? p : p.substr(d + 1);
}
static bool glob_rec(const std::vector<std::string>& pat, size_t i, const std::vector<std::string>& con, size_t j) {
    if (i == pat.size()) return j == con.size();
    if (pat[i] == "**") {
        for (size_t t = j; t <= con.size(); ++t)
            if (glob_rec(pat, i + 1, con, t)) return true;
        return false;
    }
    if (j == con.size()) return false;
    if (pat[i] != "*" && pat[i] != con[j]) return false;
    return glob_rec(pat, i + 1, con, j + 1);
}
bool glob_match(const std::string& pattern, const std::string& concrete) {
    return glob_rec(split_path(pattern), 0, split_path(concrete), 0);
}
bool has_glob(const std::string& p) {
    for (auto& s : split_path(p))
        if (s == "*" || s == "**") return true;
    return false;
}
std::vector<std::string> all_module_paths(const Module& root) {
    std::vector<std::string> out;
    std::function<void(const Module&, const std::string&)> rec = [&](const Module& m, const std::string& p) {
        out.push_back(p);
        for (auto& c : m.children) rec(*c.mod, join(p, c.name));
    };
    rec(root, "");
    std::sort(out.begin(), out.end());
    return out;
}
std::vector<std::string> expand_glob(const Module& root, const std::string& pattern) {
    if (!has_glob(pattern)) return root.resolve(pattern) ? std::vector<std::string>{pattern} : std::vector<std::string>{};
    std::vector<std::string> out;
    for (auto& p : all_module_paths(root))
        if (!p.empty() && glob_match(pattern, p)) out.push_back(p);
    return out;
}

// ------------------------------------------------------- builtin modules
Module make_linear(i64 in, i64 out, bool bias, u64 seed) {
    Module m;
    m.kind = "Linear";
    m.attrs["in_features"] = in;
    m.attrs["out_features"] = out;
    Param w;
    w.name = "weight";
    w.spec.shape = {out, in};  // out-major
    w.init = Init::Normal;
    w.seed = seed;
    m.params.push_back(w);
    if (bias) {
        Param b;
        b.name = "bias";
        b.spec.shape = {out};
        b.init = Init::Zeros;
        b.seed = seed + 1;
        m.params.push_back(b);
    }
    return m;
}
Module make_layernorm(i64 n, double eps, u64 seed) {
    Module m;
    m.kind = "LayerNorm";
    m.attrs["normalized_size"] = n;
    m.attrs["eps"] = eps;
    Param g, b;
    g.name = "gamma";
    g.spec.shape = {n};
    g.init = Init::Ones;
    g.seed = seed;
    b.name = "beta";
    b.spec.shape = {n};
    b.init = Init::Zeros;
    b.seed = seed + 1;
    m.params = {g, b};
    return m;
}
Module make_dropout(double p, u64 seed) {
    Module m;
    m.kind = "Dropout";
    m.attrs["p"] = p;
    m.attrs["seed"] = (i64)seed;
    return m;
}
Module make_embedding(i64 rows, i64 dim, u64 seed) {
    Module m;
    m.kind = "Embedding";
    m.attrs["num_embeddings"] = rows;
    m.attrs["dim"] = dim;
    Param w;
    w.name = "weight";
    w.spec.shape = {rows, dim};
    w.init = Init::Normal;
    w.seed = seed;
    m.params.push_back(w);
    return m;
}

// ------------------------------------------------- param materialisation
// Value of the full (unsharded) parameter at flat index i. A pure function of
// (init, seed, i), so any shard can be generated without the full tensor.
static double plain_value(Init init, u64 seed, i64 i) {
    switch (init) {
        case Init::Normal: return 0.1 * normal01(seed, 0x9a7a, (u64)i);
        case Init::Uniform: return 0.2 * uniform01(seed, 0x9a7b, (u64)i) - 0.1;
        case Init::Zeros: return 0.0;
        case Init::Ones: return 1.0;
    }
    return 0.0;
}

static double param_value(const Param& p, i64 full_numel, i64 i) {
    double v;
    if (!p.values.empty()) {
        v = p.values[(size_t)i];
    } else if (p.block_seeds.empty()) {
        v = plain_value(p.init, p.seed, i);
    } else {
        i64 blocks = (i64)p.block_seeds.size(), per = full_numel / blocks;
        v = plain_value(p.init, p.block_seeds[(size_t)(i / per)], i % per);
    }
    return p.spec.dtype == Dtype::F32 ? (double)(float)v : v;
}

static void check_param(const Param& p, i64 full_numel) {
    if (!p.values.empty() && (i64)p.values.size() != full_numel)
        throw Error("param '" + p.name + "' has " + std::to_string(p.values.size()) +
                    " explicit values for shape with " + std::to_string(full_numel) + " elements");
    if (p.values.empty() && !p.block_seeds.empty()) {
        auto fs = p.full_shape();
        if (fs.empty() || fs[0] % (i64)p.block_seeds.size() != 0)
            throw Error("param '" + p.name + "' rows not divisible into " + std::to_string(p.block_seeds.size()) + " blocks");
    }
}

// local flat index -> full flat index for rank `rank` of a (block-)sharded param
// (proj/src/module.cpp:435-498).
void shard_index_map(const Param& p, int rank, std::vector<i64>& out) {
    std::vector<i64> full = p.full_shape();
    i64 n_full = 1;
    for (i64 d : full) n_full *= d;
    if (!p.shard) {
        out.resize((size_t)n_full);
        for (i64 i = 0; i < n_full; ++i) out[(size_t)i] = i;
        return;
    }
    int axis = p.shard->axis, world = p.shard->world, blocks = std::max(1, p.shard->blocks);
    if (axis < 0 || axis >= (int)full.size())
        throw Error("shard axis " + std::to_string(axis) + " out of range for rank-" + std::to_string(full.size()) + " tensor");
    i64 dim = full[(size_t)axis];
    if (dim % blocks != 0) throw Error("dimension " + std::to_string(dim) + " not divisible into " + std::to_string(blocks) + " blocks");
    i64 group = dim / blocks;
    if (group % world != 0)
        throw Error((blocks > 1 ? "block dimension " : "dimension ") + std::to_string(group) +
                    " not divisible by world size " + std::to_string(world));
    i64 part = group / world, inner = 1, outer = 1;
    for (size_t i = (size_t)axis + 1; i < full.size(); ++i) inner *= full[i];
    for (int i = 0; i < axis; ++i) outer *= full[(size_t)i];
    out.resize((size_t)(outer * part * blocks * inner));
    size_t k = 0;
    for (i64 o = 0; o < outer; ++o)
        for (int b = 0; b < blocks; ++b)
            for (i64 a = 0; a < part; ++a) {
                i64 src = (o * dim + b * group + (i64)rank * part + a) * inner;
                for (i64 x = 0; x < inner; ++x) out[k++] = src + x;
            }
}

static void parallel_for(i64 n, const std::function<void(i64, i64)>& f) {
    unsigned hw = std::max(1u, std::thread::hardware_concurrency());
    if (n < (1 << 16) || hw == 1) {
        f(0, n);
        return;
    }
    unsigned nt = std::min<unsigned>(hw, 32);
    std::vector<std::thread> ts;
    i64 chunk = (n + nt - 1) / nt;
    for (unsigned t = 0; t < nt; ++t) {
        i64 lo = t * chunk, hi = std::min(n, lo + chunk);
        if (lo < hi) ts.emplace_back(f, lo, hi);
    }
    for (auto& t : ts) t.join();
}

HostTensor param_full(const Param& p) {
    TensorSpec s;
    s.shape = p.full_shape();
    s.dtype = p.spec.dtype;
    HostTensor t(s);
    i64 n = s.numel();
    check_param(p, n);
    parallel_for(n, [&](i64 lo, i64 hi) {
        for (i64 i = lo; i < hi; ++i) t.data[(size_t)i] = param_value(p, n, i);
    });
    return t;
}

HostTensor param_rank(const Param& p, int rank) {
    std::vector<i64> map;
    shard_index_map(p, rank, map);
    TensorSpec s = p.spec;
    if (p.shard) {
        s.shape = p.full_shape();
        int blocks = std::max(1, p.shard->blocks);
        s.shape[(size_t)p.shard->axis] = s.shape[(size_t)p.shard->axis] / blocks / p.shard->world * blocks;
    }
    HostTensor t(s);
    i64 n_full = 1;
    for (i64 d : p.full_shape()) n_full *= d;
    check_param(p, n_full);
    parallel_for((i64)map.size(), [&](i64 lo, i64 hi) {
        for (i64 i = lo; i < hi; ++i) t.data[(size_t)i] = param_value(p, n_full, map[(size_t)i]);
    });
    return t;
}

HostTensor slice_axis(const HostTensor& full, int axis, int world, int rank) {
    auto& sh = full.spec.shape;
    if (axis < 0 || axis >= (int)sh.size())
        throw Error("shard axis " + std::to_string(axis) + " out of range for rank-" + std::to_string(sh.size()) + " tensor");
    if (sh[(size_t)axis] % world != 0)
        throw Error("dimension " + std::to_string(sh[(size_t)axis]) + " not divisible by world size " + std::to_string(world));
    i64 part = sh[(size_t)axis] / world, inner = 1, outer = 1;
    for (size_t i = (size_t)axis + 1; i < sh.size(); ++i) inner *= sh[i];
    for (int i = 0; i < axis; ++i) outer *= sh[(size_t)i];
    TensorSpec ls = full.spec;
    ls.shape[(size_t)axis] = part;
    HostTensor out(ls);
    size_t k = 0;
    for (i64 o = 0; o < outer; ++o)
        for (i64 a = 0; a < part; ++a)
            for (i64 x = 0; x < inner; ++x) out.data[k++] = full.data[(size_t)((o * sh[(size_t)axis] + rank * part + a) * inner + x)];
    return out;
}

// -------------------------------------------------------- shape inference
bool is_builtin_op(const std::string& op) {
    static const std::set<std::string> s = {"matmul",  "add",    "mul",     "scale",      "transpose", "reshape",
                                            "split",   "concat", "relu",    "gelu",       "softmax",   "layernorm",
                                            "dropout", "reduce_sum", "all_reduce", "all_gather"};
    return s.count(op) > 0;
}

[[noreturn]] static void shape_fail(int id, const std::string& d) {
    throw Error("shape mismatch at node " + std::to_string(id) + ": " + d);
}
static int norm_axis(i64 axis, int rank, int id) {
    i64 a = axis < 0 ? axis + rank : axis;
    if (a < 0 || a >= rank) shape_fail(id, "axis " + std::to_string(axis) + " out of range for rank " + std::to_string(rank));
    return (int)a;
}
static const TensorSpec& one_arg(const std::vector<const ValueSpec*>& a, size_t i, int id) {
    if (i >= a.size()) shape_fail(id, "missing operand " + std::to_string(i));
    if (a[i]->tuple) shape_fail(id, "operand " + std::to_string(i) + " is a tuple");
    return a[i]->parts[0];
}

ValueSpec infer_op(const std::string& op, const std::vector<const ValueSpec*>& args, const Attrs& at, int id) {
    if (op == "matmul") {
        const TensorSpec &a = one_arg(args, 0, id), &b = one_arg(args, 1, id);
        if (a.rank() < 2 || b.rank() < 2)
            shape_fail(id, "matmul needs rank >= 2 operands, got " + a.str() + " and " + b.str());
        if (a.rank() != b.rank()) shape_fail(id, "matmul rank mismatch: " + a.str() + " vs " + b.str());
        for (int i = 0; i < a.rank() - 2; ++i)
            if (a.shape[(size_t)i] != b.shape[(size_t)i]) shape_fail(id, "matmul batch dims differ: " + a.str() + " vs " + b.str());
        if (a.shape.back() != b.shape[(size_t)b.rank() - 2])
            shape_fail(id, "matmul contraction mismatch between " + a.str() + " and " + b.str());
        TensorSpec o = a;
        o.shape.back() = b.shape.back();
        return ValueSpec(o);
    }
    if (op == "add" || op == "mul") {
        const TensorSpec &a = one_arg(args, 0, id), &b = one_arg(args, 1, id);
        if (a.shape.empty()) return ValueSpec(b);
        if (b.shape.empty()) return ValueSpec(a);
        if (a.shape != b.shape) shape_fail(id, "operand shapes differ: " + a.str() + " vs " + b.str());
        return ValueSpec(a);
    }
    if (op == "scale" || op == "relu" || op == "gelu" || op == "dropout" || op == "all_reduce")
        return ValueSpec(one_arg(args, 0, id));
    if (op == "softmax" || op == "layernorm") {
        const TensorSpec& x = one_arg(args, 0, id);
        norm_axis(get_int(at, "axis").value_or(-1), std::max(x.rank(), 1), id);
        return ValueSpec(x);
    }
    if (op == "transpose") {
        const TensorSpec& x = one_arg(args, 0, id);
        TensorSpec o = x;
        if (auto perm = get_ints(at, "perm")) {
            if ((int)perm->size() != x.rank()) shape_fail(id, "perm length != rank of " + x.str());
            std::vector<bool> seen((size_t)x.rank(), false);
            for (int i = 0; i < x.rank(); ++i) {
                int p = norm_axis((*perm)[(size_t)i], x.rank(), id);
                if (seen[(size_t)p]) shape_fail(id, "perm repeats axis");
                seen[(size_t)p] = true;
                o.shape[(size_t)i] = x.shape[(size_t)p];
            }
            return ValueSpec(o);
        }
        auto axes = get_ints(at, "axes").value_or(std::vector<i64>{-2, -1});
        if (axes.size() != 2) shape_fail(id, "transpose axes expects two entries");
        if (x.rank() < 2) shape_fail(id, "transpose needs rank >= 2, got " + x.str());
        std::swap(o.shape[(size_t)norm_axis(axes[0], x.rank(), id)], o.shape[(size_t)norm_axis(axes[1], x.rank(), id)]);
        return ValueSpec(o);
    }
    if (op == "reshape") {
        const TensorSpec& x = one_arg(args, 0, id);
        TensorSpec o = x;
        if (auto shape = get_ints(at, "shape")) {
            o.shape = *shape;
            int inf = -1;
            i64 prod = 1;
            for (size_t i = 0; i < o.shape.size(); ++i) {
                if (o.shape[i] == -1) {
                    if (inf >= 0) shape_fail(id, "reshape allows one -1 dim");
                    inf = (int)i;
                } else {
                    prod *= o.shape[i];
                }
            }
            if (inf >= 0) {
                if (prod == 0 || x.numel() % prod != 0) shape_fail(id, "cannot infer -1 dim reshaping " + x.str());
                o.shape[(size_t)inf] = x.numel() / prod;
            }
            if (o.numel() != x.numel()) shape_fail(id, "reshape element count differs: " + x.str() + " -> " + o.str());
            return ValueSpec(o);
        }
        if (auto sa = get_int(at, "split_axis")) {
            auto f = get_int(at, "factor");
            if (!f) shape_fail(id, "reshape split_axis requires factor attr");
            int a = norm_axis(*sa, x.rank(), id);
            if (x.shape[(size_t)a] % *f != 0)
                shape_fail(id, "dim " + std::to_string(x.shape[(size_t)a]) + " not divisible by factor " + std::to_string(*f));
            o.shape[(size_t)a] = x.shape[(size_t)a] / *f;
            o.shape.insert(o.shape.begin() + a + 1, *f);
            return ValueSpec(o);
        }
        if (auto mg = get_ints(at, "merge_axes")) {
            if (mg->size() != 2) shape_fail(id, "merge_axes expects two adjacent axes");
            int a = norm_axis((*mg)[0], x.rank(), id), b = norm_axis((*mg)[1], x.rank(), id);
            if (b != a + 1) shape_fail(id, "merge_axes expects adjacent axes");
            o.shape[(size_t)a] = x.shape[(size_t)a] * x.shape[(size_t)b];
            o.shape.erase(o.shape.begin() + b);
            return ValueSpec(o);
        }
        shape_fail(id, "reshape needs shape, split_axis or merge_axes attr");
    }
    if (op == "split") {
        const TensorSpec& x = one_arg(args, 0, id);
        int axis = norm_axis(get_int(at, "axis").value_or(-1), x.rank(), id);
        std::vector<TensorSpec> parts;
        if (auto sizes = get_ints(at, "sizes")) {
            i64 tot = 0;
            for (i64 s : *sizes) tot += s;
            if (tot != x.shape[(size_t)axis])
                shape_fail(id, "split sizes sum to " + std::to_string(tot) + " but dim is " + std::to_string(x.shape[(size_t)axis]));
            for (i64 s : *sizes) {
                TensorSpec p = x;
                p.shape[(size_t)axis] = s;
                parts.push_back(p);
            }
        } else if (auto n = get_int(at, "parts")) {
            if (*n < 1 || x.shape[(size_t)axis] % *n != 0)
                shape_fail(id, "dim " + std::to_string(x.shape[(size_t)axis]) + " not divisible into " + std::to_string(*n) + " parts");
            for (i64 i = 0; i < *n; ++i) {
                TensorSpec p = x;
                p.shape[(size_t)axis] /= *n;
                parts.push_back(p);
            }
        } else {
            shape_fail(id, "split needs parts or sizes attr");
        }
        return ValueSpec::of_tuple(parts);
    }
    if (op == "concat") {
        if (args.empty()) shape_fail(id, "concat needs at least one operand");
        TensorSpec first = one_arg(args, 0, id), o = first;
        int axis = norm_axis(get_int(at, "axis").value_or(-1), first.rank(), id);
        for (size_t i = 1; i < args.size(); ++i) {
            const TensorSpec& s = one_arg(args, i, id);
            if (s.rank() != first.rank()) shape_fail(id, "concat rank mismatch: " + first.str() + " vs " + s.str());
            for (int d = 0; d < s.rank(); ++d)
                if (d != axis && s.shape[(size_t)d] != first.shape[(size_t)d])
                    shape_fail(id, "concat shapes differ off-axis: " + first.str() + " vs " + s.str());
            o.shape[(size_t)axis] += s.shape[(size_t)axis];
        }
        return ValueSpec(o);
    }
    if (op == "reduce_sum") {
        const TensorSpec& x = one_arg(args, 0, id);
        TensorSpec o = x;
        if (auto ax = get_int(at, "axis"))
            o.shape.erase(o.shape.begin() + norm_axis(*ax, x.rank(), id));
        else
            o.shape.clear();
        return ValueSpec(o);
    }
    if (op == "all_gather") {
        const TensorSpec& x = one_arg(args, 0, id);
        TensorSpec o = x;
        o.shape[(size_t)norm_axis(get_int(at, "axis").value_or(-1), x.rank(), id)] *= get_int(at, "world").value_or(1);
        return ValueSpec(o);
    }
    throw Error("unknown op '" + op + "' at node " + std::to_string(id));
}

int module_arity(const Module& m) {
    if (m.composite()) return (int)m.forward->inputs.size();
    if (m.kind == "EfficientAttention") return 3;
    return 1;
}

ValueSpec module_out_spec(const Module& m, const std::vector<TensorSpec>& ins) {
    if ((int)ins.size() != module_arity(m))
        throw Error("module '" + m.name + "' expects " + std::to_string(module_arity(m)) + " inputs, got " +
                    std::to_string(ins.size()));
    const std::string& k = m.kind;
    if (k == "Linear" || k == "FusedQKV") {
        const Param* w = m.param("weight");
        if (!w) throw Error("module '" + m.name + "' missing weight param");
        const TensorSpec& x = ins[0];
        i64 of = w->spec.shape[0], inf = w->spec.shape[1];
        if (x.rank() < 1 || x.shape.back() != inf)
            throw Error("shape mismatch at module '" + m.name + "': input " + x.str() + " does not match weight " + w->spec.str());
        TensorSpec o = x;
        o.shape.back() = of;
        if (k == "Linear") return ValueSpec(o);
        if (of % 3 != 0) throw Error("FusedQKV weight rows must divide by 3, got " + std::to_string(of));
        o.shape.back() = of / 3;
        return ValueSpec::of_tuple({o, o, o});
    }
    if (k == "LayerNorm") {
        const Param* g = m.param("gamma");
        if (g && (ins[0].rank() < 1 || ins[0].shape.back() != g->spec.shape[0]))
            throw Error("shape mismatch at module '" + m.name + "': input " + ins[0].str() +
                        " does not match normalized size " + std::to_string(g->spec.shape[0]));
        return ValueSpec(ins[0]);
    }
    if (k == "Dropout") return ValueSpec(ins[0]);
    if (k == "Embedding") {
        const Param* w = m.param("weight");
        if (!w) throw Error("module '" + m.name + "' missing weight param");
        TensorSpec o = ins[0];
        o.shape.push_back(w->spec.shape[1]);
        o.dtype = w->spec.dtype;
        return ValueSpec(o);
    }
    if (k == "EfficientAttention") {
        if (ins[0] != ins[1] || ins[0] != ins[2])
            throw Error("shape mismatch at module '" + m.name + "': q/k/v specs differ: " + ins[0].str() + ", " +
                        ins[1].str() + ", " + ins[2].str());
        if (ins[0].rank() < 2) throw Error("EfficientAttention expects rank >= 2 inputs, got " + ins[0].str());
        return ValueSpec(ins[0]);
    }
    auto mp = infer_graph(*m.forward, ins, m);
    const Node& o = m.forward->out_node();
    if (o.args.size() == 1 && !mp.at(o.args[0]).tuple) return mp.at(o.args[0]);
    std::vector<TensorSpec> parts;
    for (int a : o.args) {
        if (mp.at(a).tuple) throw Error("module '" + m.name + "' output flattens a tuple result");
        parts.push_back(mp.at(a).parts[0]);
    }
    return ValueSpec::of_tuple(parts);
}

std::map<int, ValueSpec> infer_graph(const Graph& g, const std::vector<TensorSpec>& ins, const Module& ctx) {
    if (ins.size() != g.inputs.size())
        throw Error("expected " + std::to_string(g.inputs.size()) + " inputs, got " + std::to_string(ins.size()));
    std::map<int, ValueSpec> mp;
    size_t next = 0;
    for (auto& n : g.nodes) {
        switch (n.kind) {
            case NK::Input: mp[n.id] = ValueSpec(ins[next++]); break;
            case NK::ParamRef: {
                const Param* p = ctx.resolve_param(n.target);
                if (!p) throw Error("unknown param '" + n.target + "' at node " + std::to_string(n.id));
                mp[n.id] = ValueSpec(p->spec);
                break;
            }
            case NK::CallOp: {
                std::vector<const ValueSpec*> a;
                for (int x : n.args) a.push_back(&mp.at(x));
                mp[n.id] = infer_op(n.op, a, n.attrs, n.id);
                break;
            }
            case NK::CallModule: {
                const Module* s = ctx.resolve(n.target);
                if (!s) throw Error("unknown submodule '" + n.target + "' at node " + std::to_string(n.id));
                std::vector<TensorSpec> si;
                for (int x : n.args) {
                    if (mp.at(x).tuple) throw Error("shape mismatch at node " + std::to_string(n.id) + ": tuple passed as module input");
                    si.push_back(mp.at(x).parts[0]);
                }
                mp[n.id] = module_out_spec(*s, si);
                break;
            }
            case NK::GetItem: {
                const ValueSpec& v = mp.at(n.args[0]);
                i64 idx = get_int(n.attrs, "index").value_or(0);
                if (!v.tuple || idx < 0 || idx >= (i64)v.parts.size())
                    throw Error("shape mismatch at node " + std::to_string(n.id) + ": get_item index " + std::to_string(idx) +
                                " invalid for " + v.str());
                mp[n.id] = ValueSpec(v.parts[(size_t)idx]);
                break;
            }
            case NK::Output: {
                std::vector<TensorSpec> parts;
                bool anyt = false;
                for (int x : n.args) {
                    anyt |= mp.at(x).tuple;
                    for (auto& p : mp.at(x).parts) parts.push_back(p);
                }
                mp[n.id] = (n.args.size() == 1 && !anyt) ? ValueSpec(parts[0]) : ValueSpec::of_tuple(parts);
                break;
            }
        }
    }
    return mp;
}

std::vector<TensorSpec> declared_inputs(const Graph& g) {
    std::vector<TensorSpec> out;
    for (int id : g.inputs) {
        const Node& n = g.at(id);
        auto sh = get_ints(n.attrs, "shape");
        if (!sh) throw Error("input node " + std::to_string(id) + " has no declared shape");
        TensorSpec s;
        s.shape = *sh;
        s.dtype = dtype_from(get_str(n.attrs, "dtype").value_or("f64"));
        out.push_back(s);
    }
    return out;
}

// Input specs of the module at `path`, from the root's declared inputs down
// to its first call site (proj/src/pipeline.cpp:304-340).
std::vector<TensorSpec> module_input_specs_at(const Module& root, const std::string& path) {
    if (path.empty()) return declared_inputs(*root.forward);
    std::vector<TensorSpec> res;
    bool found = false;
    std::function<void(const Module&, const std::string&, const std::vector<TensorSpec>&)> search =
        [&](const Module& m, const std::string& p, const std::vector<TensorSpec>& ins) {
            if (found || !m.forward) return;
            auto shapes = infer_graph(*m.forward, ins, m);
            for (auto& n : m.forward->nodes) {
                if (found) return;
                if (n.kind != NK::CallModule) continue;
                std::string full = join(p, n.target);
                std::vector<TensorSpec> si;
                for (int a : n.args) si.push_back(shapes.at(a).one());
                if (full == path) {
                    res = si;
                    found = true;
                    return;
                }
                if (path.rfind(full + ".", 0) == 0) {
                    const Module* s = m.resolve(n.target);
                    if (s && s->composite()) search(*s, full, si);
                }
            }
        };
    search(root, "", declared_inputs(*root.forward));
    if (!found) throw Error("module '" + path + "' is never called; cannot infer its inputs");
    return res;
}

HostTensor random_tensor(const TensorSpec& spec, u64 seed, u64 stream) {
    HostTensor t(spec);
    for (i64 i = 0; i < spec.numel(); ++i) t.data[(size_t)i] = normal01(seed, stream, (u64)i);
    t.round_f32();
    return t;
}

i64 embedding_row(double raw, i64 rows) {
    i64 i = (i64)std::llround(raw) % rows;
    return i < 0 ? i + rows : i;
}

}  // namespace sb
