// Schedule primitives, tracer, subgraph matcher and library replacements.
// Semantics follow the reference so that apply() produces a structurally
// identical ModuleDef (checked in tests against the compiled reference):
//   tracer          proj/src/tracer.cpp:25-170
//   matcher         proj/src/pattern.cpp:52-221
//   library         proj/src/library.cpp:9-115
//   extract_region  proj/src/schedule.cpp:58-192
//   sync lowering   proj/src/schedule.cpp:205-309
//   rules + replay  proj/src/schedule.cpp:352-559, apply :719-746
#include <algorithm>
#include <cmath>
#include <functional>
#include <set>
#include <sstream>
#include <unordered_map>
#include <unordered_set>

#include "schedule.hpp"

namespace sb {

// ====================================================================== tracer
void check_param_aliasing(const Module& root, const std::string& owner) {
    std::function<void(const Module&, const std::string&)> walk = [&](const Module& m, const std::string& path) {
        if (m.forward) {
            for (auto& n : m.forward->nodes) {
                if (n.kind != NK::ParamRef) continue;
                std::string full = join(path, parent_of(n.target));
                bool inside = full == owner || full.rfind(owner + ".", 0) == 0;
                bool from_inside = path == owner || path.rfind(owner + ".", 0) == 0;
                bool from_parent = owner.rfind(path.empty() ? "" : path + ".", 0) == 0 && (path.empty() || owner != path);
                if (inside && !from_inside && !from_parent)
                    throw Error("parameter aliasing across inlined boundary is unsupported: '" + join(path, n.target) + "'");
            }
        }
        for (auto& c : m.children) walk(*c.mod, join(path, c.name));
    };
    walk(root, "");
}

Graph inline_call(const Graph& g, int call_node, const Graph& callee, const std::string& prefix) {
    const Node& call = g.at(call_node);
    if (call.kind != NK::CallModule) throw Error("inline target node " + std::to_string(call_node) + " is not call_module");
    if (call.args.size() != callee.inputs.size())
        throw Error("arity mismatch inlining '" + prefix + "': call has " + std::to_string(call.args.size()) +
                    " args, callee expects " + std::to_string(callee.inputs.size()));
    Graph out;
    out.inputs = g.inputs;
    int next = std::max(g.max_id(), callee.max_id()) + 1;
    std::unordered_map<int, int> cmap, alias;
    std::vector<int> results;
    for (auto& n : g.nodes) {
        if (n.id != call_node) {
            Node c = n;
            for (auto& a : c.args) {
                auto it = alias.find(a);
                if (it != alias.end()) a = it->second;
            }
            out.nodes.push_back(std::move(c));
            continue;
        }
        size_t in_i = 0;
        for (auto& cn : callee.nodes) {
            if (cn.kind == NK::Input) {
                cmap[cn.id] = call.args[in_i++];
                continue;
            }
            if (cn.kind == NK::Output) {
                for (int r : cn.args) results.push_back(cmap.at(r));
                continue;
            }
            Node c = cn;
            c.id = next++;
            for (auto& a : c.args) a = cmap.at(a);
            if (c.kind == NK::ParamRef || c.kind == NK::CallModule) c.target = join(prefix, c.target);
            cmap[cn.id] = c.id;
            out.nodes.push_back(std::move(c));
        }
        alias[call_node] = results.size() == 1 ? results[0] : -1;
    }
    if (results.size() > 1) {
        std::unordered_map<int, int> item;
        Graph fixed;
        fixed.inputs = out.inputs;
        for (auto& n : out.nodes) {
            if (n.kind == NK::GetItem && n.args[0] == -1) {
                i64 idx = get_int(n.attrs, "index").value_or(0);
                if (idx < 0 || idx >= (i64)results.size()) throw Error("get_item index out of range after inlining");
                item[n.id] = results[(size_t)idx];
                continue;
            }
            Node c = n;
            for (auto& a : c.args) {
                auto it = item.find(a);
                if (it != item.end()) a = it->second;
                if (a == -1) throw Error("multi-result inlined call used without get_item");
            }
            fixed.nodes.push_back(std::move(c));
        }
        out = std::move(fixed);
    } else {
        for (auto& n : out.nodes)
            for (auto& a : n.args) {
                auto it = alias.find(a);
                if (it != alias.end()) a = it->second;
            }
    }
    out.out = out.nodes.back().id;
    out.validate();
    return out;
}

static bool matches_any(const std::vector<std::string>& pats, const std::string& rel) {
    for (auto& p : pats)
        if (glob_match(p, rel)) return true;
    return false;
}

int flatten_module(Module& t, const TraceSpec& spec, std::vector<std::string>* warnings) {
    if (!t.composite()) throw Error("cannot trace builtin module '" + t.name + "'");
    if (warnings)
        for (auto& l : spec.leaves)
            if (expand_glob(t, l).empty()) warnings->push_back("leaf pattern '" + l + "' matches nothing");
    if (!spec.flatten) return 0;
    int inlined = 0;
    for (bool changed = true; changed;) {
        changed = false;
        for (auto& n : t.forward->nodes) {
            if (n.kind != NK::CallModule) continue;
            const Module* s = t.resolve(n.target);
            if (!s) throw Error("unknown submodule '" + n.target + "'");
            if (!s->composite() || matches_any(spec.leaves, n.target)) continue;
            t.forward = inline_call(*t.forward, n.id, *s->forward, n.target);
            ++inlined;
            changed = true;
            break;
        }
    }
    return inlined;
}

// ===================================================================== matcher
static bool is_core(const Node& n) { return n.kind != NK::Input && n.kind != NK::Output; }

static std::string graph_label(const Node& n, const Module* host) {
    switch (n.kind) {
        case NK::CallOp: return "op:" + n.op;
        case NK::CallModule: {
            if (host)
                if (const Module* m = host->resolve(n.target)) return "mod:" + m->kind;
            return "mod:" + n.target;
        }
        case NK::ParamRef: return "param";
        case NK::GetItem: return "get_item";
        default: return nk_str(n.kind);
    }
}
static std::string pattern_label(const Node& n) {
    switch (n.kind) {
        case NK::CallOp: return "op:" + n.op;
        case NK::CallModule: return "mod:" + n.target;  // pattern targets name a module kind
        case NK::ParamRef: return "param";
        case NK::GetItem: return "get_item";
        default: return nk_str(n.kind);
    }
}

std::vector<int> escaping_values(const Graph& g, const std::vector<int>& nodes) {
    std::unordered_set<int> in(nodes.begin(), nodes.end());
    std::set<int> esc;
    for (auto& n : g.nodes) {
        bool outside = !in.count(n.id);
        for (int a : n.args)
            if (in.count(a) && (outside || n.kind == NK::Output)) esc.insert(a);
    }
    return {esc.begin(), esc.end()};
}

void validate_pattern(const Graph& p) {
    p.validate();
    std::vector<int> core;
    for (auto& n : p.nodes)
        if (is_core(n)) core.push_back(n.id);
    if (core.empty()) throw Error("malformed pattern: no core nodes");
    std::unordered_set<int> cs(core.begin(), core.end());
    std::unordered_map<int, std::vector<int>> adj;
    for (auto& n : p.nodes) {
        if (!cs.count(n.id)) continue;
        for (int a : n.args)
            if (cs.count(a)) {
                adj[n.id].push_back(a);
                adj[a].push_back(n.id);
            }
    }
    std::unordered_set<int> seen;
    std::vector<int> st = {core[0]};
    while (!st.empty()) {
        int v = st.back();
        st.pop_back();
        if (!seen.insert(v).second) continue;
        for (int w : adj[v]) st.push_back(w);
    }
    if (seen.size() != cs.size()) throw Error("malformed pattern: core nodes are not connected");
}

std::vector<Match> find_matches(const Graph& g, const Graph& pat, const Module* host) {
    validate_pattern(pat);
    std::vector<const Node*> core;
    std::unordered_set<int> binders;
    for (auto& n : pat.nodes) {
        if (is_core(n)) core.push_back(&n);
        else if (n.kind == NK::Input) binders.insert(n.id);
    }
    std::unordered_map<int, int> assign, bind;
    std::unordered_set<int> used;
    std::vector<std::map<int, int>> results;
    std::function<void(size_t)> extend = [&](size_t pos) {
        if (pos == core.size()) {
            results.emplace_back(assign.begin(), assign.end());
            return;
        }
        const Node& p = *core[pos];
        std::string want = pattern_label(p);
        for (auto& gn : g.nodes) {
            if (!is_core(gn) || used.count(gn.id) || graph_label(gn, host) != want || p.args.size() != gn.args.size())
                continue;
            bool attrs_ok = true;
            for (auto& [k, v] : p.attrs) {
                auto it = gn.attrs.find(k);
                if (it == gn.attrs.end() || !(it->second == v)) attrs_ok = false;
            }
            if (!attrs_ok) continue;
            bool ok = true;
            std::vector<int> fresh;
            for (size_t i = 0; i < p.args.size() && ok; ++i) {
                int pa = p.args[i], ga = gn.args[i];
                if (binders.count(pa)) {
                    auto it = bind.find(pa);
                    if (it == bind.end()) {
                        bind[pa] = ga;
                        fresh.push_back(pa);
                    } else if (it->second != ga) {
                        ok = false;
                    }
                } else {
                    auto it = assign.find(pa);
                    if (it == assign.end() || it->second != ga) ok = false;
                }
            }
            if (ok) {
                assign[p.id] = gn.id;
                used.insert(gn.id);
                extend(pos + 1);
                used.erase(gn.id);
                assign.erase(p.id);
            }
            for (int f : fresh) bind.erase(f);
        }
    };
    extend(0);
    std::map<std::vector<int>, std::map<int, int>> by_image;
    for (auto& b : results) {
        std::vector<int> img;
        for (auto& [pid, gid] : b) img.push_back(gid);
        std::sort(img.begin(), img.end());
        if (escaping_values(g, img).size() != 1) continue;
        by_image.emplace(std::move(img), b);
    }
    std::vector<Match> out;
    std::unordered_set<int> taken;
    for (auto& [img, b] : by_image) {
        bool overlap = false;
        for (int id : img) overlap |= taken.count(id) > 0;
        if (overlap) continue;
        for (int id : img) taken.insert(id);
        Match m;
        m.nodes = img;
        m.binding = b;
        out.push_back(std::move(m));
    }
    return out;
}

std::vector<Match> find_module_calls(const Graph& g, const std::string& glob) {
    std::vector<Match> out;
    for (auto& n : g.nodes) {
        if (n.kind != NK::CallModule || !glob_match(glob, n.target)) continue;
        Match m;
        m.nodes = {n.id};
        m.binding[0] = n.id;
        out.push_back(std::move(m));
    }
    return out;
}

// ===================================================================== library
Module make_attention_core(i64 hd, double p, u64 seed, bool causal) {
    Module core;
    core.attrs["head_dim"] = hd;
    core.attrs["p"] = p;
    core.attrs["seed"] = (i64)seed;
    // f2 (decoder): the oracle extension's causal softmax (oracle/causal_ext.py), also
    // carried by an EfficientAttention that replaces this core (attrs are copied)
    if (causal) core.attrs["causal"] = (i64)1;
    double scale = 1.0 / std::sqrt((double)hd);
    GB b;
    int q = b.input(), k = b.input(), v = b.input();
    auto heads = [&](int x) {
        int s = b.op("reshape", {x}, {{"split_axis", (i64)2}, {"factor", hd}});
        return b.op("transpose", {s}, {{"perm", std::vector<i64>{0, 2, 1, 3}}});
    };
    int qh = heads(q), kh = heads(k), vh = heads(v);
    int kt = b.op("transpose", {kh}, {{"axes", std::vector<i64>{-2, -1}}});
    int s = b.op("matmul", {qh, kt});
    int sc = b.op("scale", {s}, {{"factor", scale}});
    Attrs smx{{"axis", (i64)-1}};
    if (causal) smx["causal"] = (i64)1;
    int a = b.op("softmax", {sc}, smx);
    int d = b.op("dropout", {a}, {{"p", p}, {"seed", (i64)seed}});
    int c = b.op("matmul", {d, vh});
    int back = b.op("transpose", {c}, {{"perm", std::vector<i64>{0, 2, 1, 3}}});
    int merged = b.op("reshape", {back}, {{"merge_axes", std::vector<i64>{2, 3}}});
    core.forward = b.finish({merged});
    return core;
}

Module attention_reference_graph(const Module& ea) {
    i64 hd = get_int(ea.attrs, "head_dim").value_or(0);
    if (hd <= 0) throw Error("EfficientAttention requires a positive head_dim attr");
    double p = get_double(ea.attrs, "p").value_or(0.0);
    i64 seed = get_int(ea.attrs, "seed").value_or(0);
    Module m = make_attention_core(hd, p, (u64)seed, get_int(ea.attrs, "causal").value_or(0) != 0);
    if (auto sc = get_double(ea.attrs, "scale")) {
        for (auto& n : m.forward->nodes)
            if (n.kind == NK::CallOp && n.op == "scale") n.attrs["factor"] = *sc;
    }
    m.attrs.clear();
    m.name = "attention_reference";
    return m;
}

Module make_qkv_composite(i64 hidden, u64 seed) {
    Module q;
    q.add_child("query", make_linear(hidden, hidden, true, seed));
    q.add_child("key", make_linear(hidden, hidden, true, seed + 10));
    q.add_child("value", make_linear(hidden, hidden, true, seed + 20));
    GB b;
    int x = b.input();
    q.forward = b.finish({b.call("query", {x}), b.call("key", {x}), b.call("value", {x})});
    return q;
}

Module build_fused_qkv(const Module& old) {
    std::vector<const Module*> lin;
    for (auto& c : old.children)
        if (c.mod->kind == "Linear") lin.push_back(c.mod.get());
    if (lin.size() != 3)
        throw Error("FusedQKV replacement expects a composite with exactly three Linear submodules, found " +
                    std::to_string(lin.size()));
    const Param* w0 = lin[0]->param("weight");
    i64 of = w0->spec.shape[0], inf = w0->spec.shape[1];
    bool bias = lin[0]->param("bias") != nullptr;
    for (auto* l : lin) {
        const Param* w = l->param("weight");
        if (w->spec.shape != w0->spec.shape || w->init != w0->init)
            throw Error("FusedQKV replacement requires identically shaped and initialized Linears");
        if ((l->param("bias") != nullptr) != bias) throw Error("FusedQKV replacement requires consistent bias usage");
        if (w->shard) throw Error("fuse the QKV weights before sharding, not after");
    }
    Module f;
    f.kind = "FusedQKV";
    f.attrs["in_features"] = inf;
    f.attrs["out_features"] = of * 3;
    Param w;
    w.name = "weight";
    w.spec.shape = {of * 3, inf};
    w.spec.dtype = w0->spec.dtype;
    w.init = w0->init;
    w.seed = w0->seed;
    for (auto* l : lin) w.block_seeds.push_back(l->param("weight")->seed);
    f.params.push_back(w);
    if (bias) {
        const Param* b0 = lin[0]->param("bias");
        Param b;
        b.name = "bias";
        b.spec.shape = {of * 3};
        b.spec.dtype = b0->spec.dtype;
        b.init = b0->init;
        b.seed = b0->seed;
        for (auto* l : lin) b.block_seeds.push_back(l->param("bias")->seed);
        f.params.push_back(b);
    }
    return f;
}

bool has_library_module(const std::string& n) { return n == "FusedQKV" || n == "EfficientAttention"; }

Module build_library_module(const std::string& n, const Module& old) {
    if (n == "FusedQKV") return build_fused_qkv(old);
    if (n == "EfficientAttention") {
        if (!get_int(old.attrs, "head_dim"))
            throw Error("EfficientAttention replacement requires a head_dim attr on the replaced module");
        Module ea;
        ea.kind = "EfficientAttention";
        ea.attrs = old.attrs;
        return ea;
    }
    throw Error("unknown library module '" + n + "'");
}

// ==================================================================== schedule
const char* prim_str(Prim p) {
    switch (p) {
        case Prim::Replace: return "replace";
        case Prim::Shard: return "shard";
        case Prim::Sync: return "sync";
        case Prim::Checkpoint: return "checkpoint";
        case Prim::Trace: return "trace";
        case Prim::Find: return "find";
        case Prim::Fuse: return "fuse";
        case Prim::PipelineSplit: return "pipeline_split";
    }
    return "?";
}

struct ScheduleState {
    Module original, shadow;
    WorldConfig world;
    std::vector<Record> log;
    std::map<std::string, Graph> patterns;
    std::vector<std::string> warnings;
    bool deferred = false;
};

namespace {

bool ancestor_or_same(const std::string& a, const std::string& b) {
    return a == b || a.empty() || b.rfind(a + ".", 0) == 0;
}

// Collapse `m` (a single-escape region of host's graph) into a new composite
// child `name` called as one node (proj/src/schedule.cpp:58-192 contract).
std::vector<TensorSpec> extract_region(Module& host, const Match& m, const std::string& name, const Attrs& extra,
                                       const std::vector<TensorSpec>& host_inputs) {
    Graph& g = *host.forward;
    std::unordered_set<int> region(m.nodes.begin(), m.nodes.end());
    auto esc = escaping_values(g, m.nodes);
    if (esc.size() != 1)
        throw Error("region has " + std::to_string(esc.size()) + " escaping values; exactly one is required");
    int escape = esc[0];
    auto shapes = infer_graph(g, host_inputs, host);
    std::vector<int> boundary;
    std::unordered_set<int> seen;
    for (auto& n : g.nodes) {
        if (!region.count(n.id)) continue;
        for (int a : n.args)
            if (!region.count(a) && seen.insert(a).second) boundary.push_back(a);
    }
    Module sub;
    sub.attrs = extra;
    Graph sg;
    std::unordered_map<int, int> re;
    int next = 0;
    for (int b : boundary) {
        if (shapes.at(b).tuple) throw Error("region boundary value is a tuple; unsupported");
        Node in;
        in.id = next++;
        in.kind = NK::Input;
        sg.inputs.push_back(in.id);
        re[b] = in.id;
        sg.nodes.push_back(std::move(in));
    }
    std::vector<TensorSpec> in_specs;
    for (int b : boundary) in_specs.push_back(shapes.at(b).parts[0]);
    std::vector<std::string> moved;
    for (auto& n : g.nodes) {
        if (!region.count(n.id)) continue;
        Node c = n;
        c.id = next++;
        for (auto& a : c.args) a = re.at(a);
        re[n.id] = c.id;
        if (n.kind == NK::ParamRef)
            throw Error("patterns may not capture param_ref nodes; the value arrives as a region input instead");
        if (n.kind == NK::CallModule) {
            std::string head = split_path(n.target).front();
            for (auto& o : g.nodes) {
                if (o.id == n.id || region.count(o.id)) continue;
                if (o.kind == NK::CallModule && split_path(o.target).front() == head)
                    throw Error("submodule '" + head + "' is called both inside and outside the matched region");
            }
            if (std::find(moved.begin(), moved.end(), head) == moved.end()) moved.push_back(head);
        }
        sg.nodes.push_back(std::move(c));
        if (n.kind == NK::CallOp && n.op == "reshape")
            if (auto f = get_int(n.attrs, "factor")) sub.attrs.emplace("head_dim", *f);
        if (n.kind == NK::CallOp && n.op == "dropout") {
            if (auto p = get_double(n.attrs, "p")) sub.attrs.emplace("p", *p);
            if (auto s = get_int(n.attrs, "seed")) sub.attrs.emplace("seed", *s);
        }
    }
    Node on;
    on.id = next++;
    on.kind = NK::Output;
    on.args = {re.at(escape)};
    sg.out = on.id;
    sg.nodes.push_back(std::move(on));
    sg.validate();
    sub.forward = std::move(sg);
    for (auto& c : moved) {
        const Module* cm = host.child(c);
        if (!cm) throw Error("region references unknown submodule '" + c + "'");
        sub.add_child(c, *cm);
    }
    host.add_child(name, std::move(sub));
    for (auto& c : moved)
        for (auto it = host.children.begin(); it != host.children.end(); ++it)
            if (it->name == c) {
                host.children.erase(it);
                break;
            }
    Graph ng;
    ng.inputs = g.inputs;
    int call_id = g.max_id() + 1, last = -1;
    for (size_t i = 0; i < g.nodes.size(); ++i)
        if (region.count(g.nodes[i].id)) last = (int)i;
    for (size_t i = 0; i < g.nodes.size(); ++i) {
        const Node& n = g.nodes[i];
        if (!region.count(n.id)) {
            Node c = n;
            for (auto& a : c.args)
                if (a == escape) a = call_id;
            ng.nodes.push_back(std::move(c));
        }
        if ((int)i == last) {
            Node call;
            call.id = call_id;
            call.kind = NK::CallModule;
            call.target = name;
            call.args = boundary;
            ng.nodes.push_back(std::move(call));
        }
    }
    ng.out = ng.nodes.back().id;
    try {
        ng.validate();
    } catch (const Error& e) {
        throw Error(std::string("region cannot be extracted as one node: ") + e.what());
    }
    host.forward = std::move(ng);
    return in_specs;
}

int name_counter(const Module& host, const std::string& base) {
    int i = 0;
    while (host.child(base + "_" + std::to_string(i))) ++i;
    return i;
}

int wrap_calls_with_all_reduce(Graph& g, const std::string& rel) {
    int count = 0;
    std::unordered_set<int> done;
    for (bool changed = true; changed;) {
        changed = false;
        for (auto& n : g.nodes) {
            if (n.kind != NK::CallModule || n.target != rel || done.count(n.id)) continue;
            int cid = n.id, nid = g.max_id() + 1;
            Graph ng;
            ng.inputs = g.inputs;
            for (auto& o : g.nodes) {
                Node c = o;
                if (o.id != cid)
                    for (auto& a : c.args)
                        if (a == cid) a = nid;
                ng.nodes.push_back(std::move(c));
                if (o.id == cid) {
                    Node ar;
                    ar.id = nid;
                    ar.kind = NK::CallOp;
                    ar.op = "all_reduce";
                    ar.args = {cid};
                    ng.nodes.push_back(std::move(ar));
                }
            }
            ng.out = ng.nodes.back().id;
            ng.validate();
            g = std::move(ng);
            done.insert(cid);
            ++count;
            changed = true;
            break;
        }
    }
    return count;
}

int lower_sync_live(Module& m, const std::string& path, const std::string& site, std::set<std::string>& visited) {
    if (!m.forward || !visited.insert(path).second) return 0;
    int wrapped = 0;
    std::set<std::string> rels, callees;
    for (auto& n : m.forward->nodes)
        if (n.kind == NK::CallModule && join(path, n.target) == site) rels.insert(n.target);
    for (auto& r : rels) wrapped += wrap_calls_with_all_reduce(*m.forward, r);
    for (auto& n : m.forward->nodes)
        if (n.kind == NK::CallModule) callees.insert(n.target);
    for (auto& t : callees) {
        Module* s = m.resolve(t);
        if (s && s->composite()) wrapped += lower_sync_live(*s, join(path, t), site, visited);
    }
    return wrapped;
}

void lower_sync_forward(Module& model, const std::string& site) {
    if (site.empty()) {
        Graph& g = *model.forward;
        Node o = g.out_node();
        Graph ng;
        ng.inputs = g.inputs;
        int next = g.max_id() + 1;
        for (auto& n : g.nodes)
            if (n.kind != NK::Output) ng.nodes.push_back(n);
        std::vector<int> res;
        for (int r : o.args) {
            Node ar;
            ar.id = next++;
            ar.kind = NK::CallOp;
            ar.op = "all_reduce";
            ar.args = {r};
            res.push_back(ar.id);
            ng.nodes.push_back(std::move(ar));
        }
        Node no;
        no.id = next++;
        no.kind = NK::Output;
        no.args = res;
        ng.out = no.id;
        ng.nodes.push_back(std::move(no));
        ng.validate();
        model.forward = std::move(ng);
        return;
    }
    std::set<std::string> visited;
    if (lower_sync_live(model, "", site, visited) == 0) throw Error("cannot place sync: no live call to '" + site + "' found");
}

bool subtree_checkpointed(const Module& m) {
    if (get_flag(m.attrs, "checkpoint")) return true;
    for (auto& c : m.children)
        if (subtree_checkpointed(*c.mod)) return true;
    return false;
}

void check_checkpoint_nesting(const Module& model, const std::string& site) {
    const Module* t = model.resolve(site);
    if (!t) throw Error("unknown module path '" + site + "'");
    if (subtree_checkpointed(*t))
        throw Error("nested checkpoint regions are rejected: '" + site + "' already contains a checkpointed module");
    std::string p = site;
    while (!p.empty()) {
        p = parent_of(p);
        const Module* a = model.resolve(p);
        if (a && get_flag(a->attrs, "checkpoint"))
            throw Error("nested checkpoint regions are rejected: ancestor '" + p + "' is checkpointed");
    }
}

std::vector<TensorSpec> site_specs(const Module& model, const std::string& site) {
    try {
        return module_input_specs_at(model, site);
    } catch (const Error& e) {
        throw RuleError("R4", std::string("cannot infer module interface: ") + e.what());
    }
}

std::vector<Match> pattern_matches(Module& site, const Record& r, const std::map<std::string, Graph>& patterns,
                                   std::vector<std::string>* warnings) {
    auto it = patterns.find(r.pattern);
    if (it == patterns.end()) throw Error("unknown pattern '" + r.pattern + "'");
    auto ms = find_matches(*site.forward, it->second, &site);
    if (ms.empty() && warnings) warnings->push_back("pattern '" + r.pattern + "' matched nothing at '" + r.site + "'");
    return ms;
}

}  // namespace

void check_record_rules(const Record& r, const std::vector<Record>& prior, const WorldConfig& w) {
    auto any = [&](auto pred) {
        for (auto& p : prior)
            if (pred(p)) return true;
        return false;
    };
    bool dist = r.prim == Prim::Shard || r.prim == Prim::Sync || r.prim == Prim::PipelineSplit;
    if (dist && w.world_size <= 1)
        throw RuleError("R2", std::string(prim_str(r.prim)) + " requires a distributed environment (world_size > 1)");
    if (r.prim == Prim::Sync &&
        !any([&](const Record& p) {
            return p.prim == Prim::Shard && (ancestor_or_same(p.site, r.site) || ancestor_or_same(r.site, p.site));
        }))
        throw RuleError("R1", "sync at '" + r.site +
                                  "' has no corresponding shard at the site, an ancestor, or within its subtree");
    bool needs_trace = r.prim == Prim::Fuse || r.prim == Prim::PipelineSplit ||
                       (r.prim == Prim::Replace && !r.pattern.empty()) ||
                       (r.prim == Prim::Checkpoint && !r.pattern.empty()) || (r.prim == Prim::Find && !r.pattern.empty());
    if (needs_trace && !any([&](const Record& p) { return p.prim == Prim::Trace && ancestor_or_same(p.site, r.site); }))
        throw RuleError("R3", std::string(prim_str(r.prim)) + " at '" + r.site + "' requires a static graph; apply trace first");
}

void apply_record(Module& model, const Record& r, const WorldConfig& w, const std::map<std::string, Graph>& patterns,
                  std::vector<std::string>* warnings) {
    Module* site = model.resolve(r.site);
    if (!site) throw Error("unknown module path '" + r.site + "'");
    switch (r.prim) {
        case Prim::Trace:
            if (!site->composite()) throw Error("cannot trace builtin module '" + r.site + "'");
            if (r.trace.flatten) check_param_aliasing(model, r.site);
            flatten_module(*site, r.trace, warnings);
            break;
        case Prim::Replace: {
            if (r.pattern.empty()) {
                if (r.site.empty()) throw Error("cannot replace the root module");
                auto specs = site_specs(model, r.site);
                Module rep = build_library_module(r.library, *site);
                ValueSpec before = module_out_spec(*site, specs), after;
                try {
                    after = module_out_spec(rep, specs);
                } catch (const Error& e) {
                    throw RuleError("R4", std::string("replacement rejects the module inputs: ") + e.what());
                }
                if (!(before == after))
                    throw RuleError("R4", "interface mismatch replacing '" + r.site + "': " + before.str() + " vs " + after.str());
                rep.name = last_of(r.site);
                model.resolve(parent_of(r.site))->replace_child(last_of(r.site), std::move(rep));
            } else {
                auto specs = site_specs(model, r.site);
                for (auto& m : pattern_matches(*site, r, patterns, warnings)) {
                    std::string name = "replaced_" + r.pattern + "_" + std::to_string(name_counter(*site, "replaced_" + r.pattern));
                    auto in_specs = extract_region(*site, m, name, {}, specs);
                    Module* ex = site->child(name);
                    Module rep = build_library_module(r.library, *ex);
                    ValueSpec before = module_out_spec(*ex, in_specs), after = module_out_spec(rep, in_specs);
                    if (!(before == after))
                        throw RuleError("R4", "interface mismatch replacing region at '" + r.site + "': " + before.str() +
                                                  " vs " + after.str());
                    rep.name = name;
                    site->replace_child(name, std::move(rep));
                }
            }
            break;
        }
        case Prim::Shard:
            for (auto& pn : r.params) {
                Param* p = site->param(pn);
                if (!p) throw Error("unknown param '" + pn + "' at '" + r.site + "'");
                if (p->shard) throw Error("param '" + pn + "' is already sharded");
                if (r.axis == 1 && p->spec.rank() == 1) {
                    if (warnings) warnings->push_back("bias '" + pn + "' kept whole under axis=1 sharding");
                    continue;
                }
                if (r.axis < 0 || r.axis >= p->spec.rank())
                    throw Error("shard axis " + std::to_string(r.axis) + " out of range for param '" + pn + "'");
                int blocks = (site->kind == "FusedQKV" && r.axis == 0) ? 3 : 1;
                i64 dim = p->spec.shape[(size_t)r.axis];
                if (dim % ((i64)blocks * w.world_size) != 0)
                    throw RuleError("R5", "dimension " + std::to_string(dim) + " of param '" + pn +
                                              "' is not divisible by world size " + std::to_string(w.world_size));
                ShardInfo si;
                si.axis = r.axis;
                si.world = w.world_size;
                si.blocks = blocks;
                si.full_shape = p->spec.shape;
                p->shard = si;
                p->spec.shape[(size_t)r.axis] = dim / w.world_size;
            }
            break;
        case Prim::Sync:
            if (r.sync_type != "forward" && r.sync_type != "backward" && r.sync_type != "both")
                throw Error("sync type must be forward, backward or both, got '" + r.sync_type + "'");
            if (r.sync_type != "forward") site->attrs["sync_backward"] = (i64)1;
            if (r.sync_type != "backward") lower_sync_forward(model, r.site);
            break;
        case Prim::Checkpoint:
            if (r.pattern.empty()) {
                check_checkpoint_nesting(model, r.site);
                site->attrs["checkpoint"] = (i64)1;
            } else {
                auto specs = site_specs(model, r.site);
                Attrs at{{"checkpoint", (i64)1}};
                for (auto& m : pattern_matches(*site, r, patterns, warnings)) {
                    std::string base = "ckpt_" + r.pattern;
                    extract_region(*site, m, base + "_" + std::to_string(name_counter(*site, base)), at, specs);
                }
            }
            break;
        case Prim::Find: break;
        case Prim::Fuse: {
            // "composed" is the reference's fuse backend (proj/src/schedule.cpp:526);
            // "sm100" is accepted as its B200 alias. Either way the executor lowers a
            // recognised region to one fused kernel and anything else op-by-op.
            if (r.backend != "composed" && r.backend != "sm100")
                throw Error("unknown backend '" + r.backend + "' (registered: composed, sm100)");
            auto specs = site_specs(model, r.site);
            Attrs at{{"fused", (i64)1}, {"backend", r.backend}};
            for (auto& m : pattern_matches(*site, r, patterns, warnings)) {
                std::string base = "fused_" + r.pattern;
                extract_region(*site, m, base + "_" + std::to_string(name_counter(*site, base)), at, specs);
            }
            break;
        }
        case Prim::PipelineSplit: {
            if (!site->forward) throw Error("pipeline_split target '" + r.site + "' has no graph");
            bool found = false;
            for (auto& n : site->forward->nodes) found |= n.kind == NK::CallModule && n.target == r.after_child;
            if (!found) throw Error("pipeline boundary not found: no call to '" + r.after_child + "' in '" + r.site + "'");
            break;
        }
    }
}

Schedule::Schedule(Module model, WorldConfig world) {
    model.validate();
    st_ = std::make_shared<ScheduleState>();
    st_->original = model;
    st_->shadow = std::move(model);
    st_->world = world;
}
Schedule Schedule::at(const std::string& p) const {
    std::string full = join(path_, p);
    if (!st_->shadow.resolve(full)) throw Error("unknown module path '" + full + "'");
    return Schedule(st_, full);
}
std::vector<std::string> Schedule::children() const {
    std::vector<std::string> out;
    for (auto& c : module().children) out.push_back(c.name);
    return out;
}
const Module& Schedule::module() const {
    const Module* m = st_->shadow.resolve(path_);
    if (!m) throw Error("schedule path '" + path_ + "' no longer resolves");
    return *m;
}
const Module& Schedule::original() const { return st_->original; }
const WorldConfig& Schedule::world() const { return st_->world; }
const std::vector<Record>& Schedule::log() const { return st_->log; }
const std::vector<std::string>& Schedule::warnings() const { return st_->warnings; }
void Schedule::set_deferred(bool d) { st_->deferred = d; }
void Schedule::record_raw(Record r) { st_->log.push_back(std::move(r)); }

void Schedule::record(Record r) {
    if (!st_->deferred) {
        check_record_rules(r, st_->log, st_->world);
        Module next = st_->shadow;  // a failing primitive mutates nothing
        apply_record(next, r, st_->world, st_->patterns, &st_->warnings);
        st_->shadow = std::move(next);
    }
    st_->log.push_back(std::move(r));
}

void Schedule::trace(TraceSpec spec) {
    Record r;
    r.prim = Prim::Trace;
    r.site = path_;
    r.trace = std::move(spec);
    record(std::move(r));
}
void Schedule::replace_with(const std::string& lib) {
    Record r;
    r.prim = Prim::Replace;
    r.site = path_;
    r.library = lib;
    record(std::move(r));
}
void Schedule::replace_at(const std::string& lib, const std::string& pattern) {
    Record r;
    r.prim = Prim::Replace;
    r.site = path_;
    r.library = lib;
    r.pattern = pattern;
    record(std::move(r));
}
void Schedule::shard(const std::vector<std::string>& params, int axis) {
    Record r;
    r.prim = Prim::Shard;
    r.site = path_;
    r.params = params;
    r.axis = axis;
    record(std::move(r));
}
void Schedule::sync(const std::string& type) {
    Record r;
    r.prim = Prim::Sync;
    r.site = path_;
    r.sync_type = type;
    record(std::move(r));
}
void Schedule::checkpoint() {
    Record r;
    r.prim = Prim::Checkpoint;
    r.site = path_;
    record(std::move(r));
}
void Schedule::checkpoint_at(const std::string& pattern) {
    Record r;
    r.prim = Prim::Checkpoint;
    r.site = path_;
    r.pattern = pattern;
    record(std::move(r));
}
std::vector<Match> Schedule::find(const std::string& glob) {
    Record r;
    r.prim = Prim::Find;
    r.site = path_;
    record(std::move(r));
    auto out = find_module_calls(*module().forward, glob);
    for (auto& m : out) m.site = path_;
    return out;
}
std::vector<Match> Schedule::find(const Graph& pattern) {
    Record r;
    r.prim = Prim::Find;
    r.site = path_;
    r.pattern = "<inline>";
    record(std::move(r));
    auto out = find_matches(*module().forward, pattern, &module());
    for (auto& m : out) m.site = path_;
    return out;
}
void Schedule::fuse_at(const std::string& pattern, const std::string& backend) {
    Record r;
    r.prim = Prim::Fuse;
    r.site = path_;
    r.pattern = pattern;
    r.backend = backend;
    record(std::move(r));
}
void Schedule::pipeline_split(const std::string& after) {
    Record r;
    r.prim = Prim::PipelineSplit;
    r.site = path_;
    r.after_child = after;
    record(std::move(r));
}
void Schedule::define_pattern(const std::string& name, Graph pattern) {
    validate_pattern(pattern);
    st_->patterns[name] = std::move(pattern);
}

ApplyResult Schedule::apply() const {
    for (size_t i = 0; i < st_->log.size(); ++i) {
        std::vector<Record> prior(st_->log.begin(), st_->log.begin() + (long)i);
        check_record_rules(st_->log[i], prior, st_->world);
    }
    ApplyResult res;
    res.model = st_->original;
    std::vector<std::string> sink;
    for (size_t i = 0; i < st_->log.size(); ++i) {
        try {
            apply_record(res.model, st_->log[i], st_->world, st_->patterns, &sink);
        } catch (const Error& e) {
            throw Error("apply failed at record " + std::to_string(i) + " (" + prim_str(st_->log[i].prim) + " at '" +
                        st_->log[i].site + "'): " + e.what());
        }
        if (st_->log[i].prim == Prim::PipelineSplit) res.pipeline_splits.push_back({st_->log[i].site, st_->log[i].after_child});
    }
    return res;
}

// ================================================================ script
namespace {
std::string strip(const std::string& s) {
    size_t a = s.find_first_not_of(" \t\r\n"), b = s.find_last_not_of(" \t\r\n");
    return a == std::string::npos ? "" : s.substr(a, b - a + 1);
}
std::string strip_comment(const std::string& s) {
    auto h = s.find('#');
    return h == std::string::npos ? s : s.substr(0, h);
}
std::vector<std::string> toks_of(const std::string& s) {
    std::istringstream is(s);
    std::vector<std::string> t;
    std::string w;
    while (is >> w) t.push_back(w);
    return t;
}
std::optional<std::string> kv(const std::string& tok, const std::string& key) {
    if (tok.rfind(key + "=", 0) == 0) return tok.substr(key.size() + 1);
    return std::nullopt;
}
std::vector<std::string> commas(const std::string& s) {
    std::vector<std::string> out;
    std::string cur;
    for (char c : s) {
        if (c == ',') {
            if (!cur.empty()) out.push_back(cur);
            cur.clear();
        } else {
            cur += c;
        }
    }
    if (!cur.empty()) out.push_back(cur);
    return out;
}
[[noreturn]] void sfail(int line, const std::string& m) { throw Error("script line " + std::to_string(line) + ": " + m); }
}  // namespace

void load_schedule_script(Schedule& s, const std::string& text) {
    s.set_deferred(true);
    const Module& model = s.original();
    std::vector<std::string> lines;
    {
        std::istringstream is(text);
        std::string l;
        while (std::getline(is, l)) lines.push_back(l);
    }
    auto sites = [&](const std::string& raw, int ln) -> std::vector<std::string> {
        std::string p = raw == "." ? "" : raw;
        if (p.empty() || !has_glob(p)) return {p};
        auto v = expand_glob(model, p);
        if (v.empty()) sfail(ln, "glob '" + raw + "' matches no modules");
        return v;
    };
    for (size_t li = 0; li < lines.size(); ++li) {
        int ln = (int)li + 1;
        std::string line = strip(strip_comment(lines[li]));
        if (line.empty()) continue;
        if (line.rfind("pattern", 0) == 0) {
            std::istringstream head(line);
            std::string kw, name, rest;
            head >> kw >> name;
            if (name.empty() || name.back() == '{') sfail(ln, "pattern needs a name");
            std::getline(head, rest);
            std::string body;
            int depth = 0;
            bool opened = false;
            size_t scan = li;
            std::string chunk = rest;
            while (true) {
                bool closed = false;
                for (char c : chunk) {
                    if (c == '{') {
                        ++depth;
                        opened = true;
                        if (depth == 1) continue;
                    }
                    if (c == '}') {
                        --depth;
                        if (depth == 0) {
                            closed = true;
                            break;
                        }
                    }
                    if (opened && depth >= 1) body += c;
                }
                if (closed) break;
                if (++scan >= lines.size()) sfail(ln, "unterminated pattern block");
                chunk = strip_comment(lines[scan]);
                body += '\n';
            }
            li = scan;
            try {
                s.define_pattern(name, parse_graph_json(strip(body)));
            } catch (const Error& e) {
                sfail(ln, std::string("bad pattern graph: ") + e.what());
            }
            continue;
        }
        auto t = toks_of(line);
        const std::string& cmd = t[0];
        Record r;
        std::vector<std::string> where;
        if (cmd == "trace") {
            if (t.size() < 2) sfail(ln, "trace needs a path");
            r.prim = Prim::Trace;
            for (size_t i = 2; i < t.size(); ++i) {
                if (auto v = kv(t[i], "flatten")) r.trace.flatten = *v == "true" || *v == "1";
                else if (auto l = kv(t[i], "leaves")) r.trace.leaves = commas(*l);
                else sfail(ln, "unknown trace option '" + t[i] + "'");
            }
            where = sites(t[1], ln);
        } else if (cmd == "replace") {
            if (t.size() < 4 || t[2] != "with") sfail(ln, "usage: replace <path> with <library-module> [at <pattern>]");
            r.prim = Prim::Replace;
            r.library = t[3];
            if (t.size() >= 6 && t[4] == "at") r.pattern = t[5];
            else if (t.size() > 4) sfail(ln, "unexpected tokens after library module");
            where = sites(t[1], ln);
        } else if (cmd == "shard") {
            if (t.size() != 4) sfail(ln, "usage: shard <path> <params> axis=<0|1>");
            auto ax = kv(t[3], "axis");
            if (!ax) sfail(ln, "shard needs axis=<0|1>");
            r.prim = Prim::Shard;
            r.params = commas(t[2]);
            r.axis = std::stoi(*ax);
            where = sites(t[1], ln);
        } else if (cmd == "sync") {
            if (t.size() != 3) sfail(ln, "usage: sync <path> type=<forward|backward|both>");
            auto ty = kv(t[2], "type");
            if (!ty) sfail(ln, "sync needs type=<forward|backward|both>");
            r.prim = Prim::Sync;
            r.sync_type = *ty;
            where = sites(t[1], ln);
        } else if (cmd == "checkpoint") {
            r.prim = Prim::Checkpoint;
            if (t.size() == 4 && t[2] == "at") r.pattern = t[3];
            else if (t.size() != 2) sfail(ln, "usage: checkpoint <path> [at <pattern>]");
            where = sites(t[1], ln);
        } else if (cmd == "fuse") {
            if (t.size() < 4 || t[2] != "at") sfail(ln, "usage: fuse <path> at <pattern> backend=<name>");
            r.prim = Prim::Fuse;
            r.pattern = t[3];
            r.backend = "composed";
            if (t.size() == 5) {
                auto b = kv(t[4], "backend");
                if (!b) sfail(ln, "expected backend=<name>");
                r.backend = *b;
            }
            where = sites(t[1], ln);
        } else if (cmd == "pipeline_split") {
            if (t.size() != 3) sfail(ln, "usage: pipeline_split <path> after=<child>");
            auto a = kv(t[2], "after");
            if (!a) sfail(ln, "pipeline_split needs after=<child-segment>");
            r.prim = Prim::PipelineSplit;
            r.after_child = *a;
            where = sites(t[1], ln);
        } else {
            sfail(ln, "unknown primitive '" + cmd + "'");
        }
        for (auto& w : where) {
            Record c = r;
            c.site = w;
            s.record_raw(std::move(c));
        }
    }
}

}  // namespace sb
