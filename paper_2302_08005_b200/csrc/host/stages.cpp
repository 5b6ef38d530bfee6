// Pipeline stage materialisation: the recorded
// pipeline_split boundaries become self-contained stage modules with named
// stage I/O, following the reference's partitioner (proj/src/pipeline.cpp
// build_pipeline_plan :343-420, segment_module :40-193, inline_parts :198-283)
// so that the stage modules serialise identically:
//   * boundaries recorded in a submodule are propagated upwards level by level
//     (deepest site first): the module is cut into sequential parts, the parts
//     replace its single call in the parent, and the parent inherits the cuts;
//   * the top module is cut into stages; a value crosses a cut when it is
//     produced before it and used at or after it (liveness by position).
#include "stages.hpp"

#include <algorithm>
#include <map>
#include <set>
#include <unordered_map>

namespace sb {

namespace {

std::string dots_to_underscores(std::string s) {
    std::replace(s.begin(), s.end(), '.', '_');
    return s;
}

std::string boundary_value_name(const Graph& g, int id) {  // pipeline.cpp:24-29
    const Node& n = g.at(id);
    if (n.kind == NK::CallModule) return "n" + std::to_string(id) + "_" + dots_to_underscores(n.target);
    if (n.kind == NK::CallOp) return "n" + std::to_string(id) + "_" + n.op;
    return "n" + std::to_string(id);
}

struct Parts {
    std::vector<Module> mods;
    std::vector<std::vector<std::string>> in_names, out_names;  // per part
    std::vector<std::string> module_inputs, module_results;
};

Parts cut_module(const Module& m, std::vector<int> cuts, const std::vector<TensorSpec>& in_specs) {
    const Graph& g = *m.forward;
    const std::map<int, ValueSpec> shapes = infer_graph(g, in_specs, m);
    std::sort(cuts.begin(), cuts.end(), [&](int a, int b) { return g.pos(a) < g.pos(b); });
    const int nparts = (int)cuts.size() + 1;

    std::unordered_map<int, int> part_of;  // node -> part, by position
    {
        size_t k = 0;
        int p = 0;
        for (auto& n : g.nodes) {
            if (n.kind == NK::Output) break;
            if (n.kind == NK::Input) continue;
            part_of[n.id] = p;
            if (k < cuts.size() && n.id == cuts[k]) ++k, ++p;
        }
    }
    std::unordered_map<int, int> made_in;  // value -> producing part (-1: module input)
    std::unordered_map<int, std::string> name;
    Parts out;
    for (size_t i = 0; i < g.inputs.size(); ++i) {
        made_in[g.inputs[i]] = -1;
        name[g.inputs[i]] = "in" + std::to_string(i);
        out.module_inputs.push_back(name[g.inputs[i]]);
    }
    for (auto& n : g.nodes)
        if (n.kind != NK::Input && n.kind != NK::Output) {
            made_in[n.id] = part_of.at(n.id);
            name[n.id] = boundary_value_name(g, n.id);
        }
    std::unordered_map<int, int> last_user;  // value -> last part reading it (results: one past the end)
    for (auto& n : g.nodes) {
        if (n.kind == NK::Input) continue;
        const int user = n.kind == NK::Output ? nparts : part_of.at(n.id);
        for (int a : n.args) {
            auto it = last_user.find(a);
            if (it == last_user.end() || it->second < user) last_user[a] = user;
        }
    }
    for (int r : g.out_node().args) out.module_results.push_back(name.at(r));

    for (int s = 0; s < nparts; ++s) {
        std::vector<int> ins, outs;
        for (auto& n : g.nodes) {
            if (n.kind == NK::Output) continue;
            const int p = made_in.at(n.id);
            auto lu = last_user.find(n.id);
            const int last = lu == last_user.end() ? -2 : lu->second;
            if (p < s && last >= s) ins.push_back(n.id);
            if (p <= s && last >= s + 1) outs.push_back(n.id);
        }
        Module part;
        part.kind = "composite";
        part.name = "part" + std::to_string(s);
        Graph pg;
        std::unordered_map<int, int> id_map;
        int next = 0;
        for (int id : ins) {
            Node in;
            in.id = next++;
            in.kind = NK::Input;
            const ValueSpec& vs = shapes.at(id);
            if (vs.tuple) throw Error("pipeline boundary value '" + name.at(id) + "' is a tuple");
            in.attrs["shape"] = vs.parts[0].shape;
            in.attrs["dtype"] = std::string(dtype_str(vs.parts[0].dtype));
            pg.inputs.push_back(in.id);
            id_map[id] = in.id;
            pg.nodes.push_back(std::move(in));
        }
        std::set<std::string> children, params;  // ordered: stage modules serialise deterministically
        for (auto& n : g.nodes) {
            if (n.kind == NK::Input || n.kind == NK::Output || part_of.at(n.id) != s) continue;
            Node c = n;
            c.id = next++;
            for (auto& a : c.args) {
                auto it = id_map.find(a);
                if (it == id_map.end()) throw Error("pipeline segmentation lost value " + std::to_string(a));
                a = it->second;
            }
            id_map[n.id] = c.id;
            if (n.kind == NK::CallModule) children.insert(split_path(n.target).front());
            if (n.kind == NK::ParamRef) {
                const std::string head = split_path(n.target).front();
                if (m.param(head) || m.param(n.target)) params.insert(n.target);
                else children.insert(head);
            }
            pg.nodes.push_back(std::move(c));
        }
        Node o;
        o.id = next++;
        o.kind = NK::Output;
        for (int id : outs) o.args.push_back(id_map.at(id));
        pg.out = o.id;
        pg.nodes.push_back(std::move(o));
        pg.validate();
        part.forward = std::move(pg);
        for (auto& c : children) {
            const Module* sub = m.child(c);
            if (!sub) throw Error("pipeline segmentation: unknown child '" + c + "'");
            part.add_child(c, *sub);
        }
        for (auto& pn : params)
            if (const Param* p = m.param(pn)) part.params.push_back(*p);
        out.mods.push_back(std::move(part));
        std::vector<std::string> in_n, out_n;
        for (int id : ins) in_n.push_back(name.at(id));
        for (int id : outs) out_n.push_back(name.at(id));
        out.in_names.push_back(std::move(in_n));
        out.out_names.push_back(std::move(out_n));
    }
    std::map<std::string, int> owner;  // a child used by two parts would alias state across stages
    for (int s = 0; s < nparts; ++s)
        for (auto& c : out.mods[(size_t)s].children) {
            auto [it, fresh] = owner.emplace(c.name, s);
            if (!fresh && it->second != s) throw Error("submodule '" + c.name + "' is used by two pipeline segments");
        }
    return out;
}

// Replace the single call to `seg` in `parent` by the chain of part calls;
// returns the part-call ids that carry the propagated cuts (all but the last).
std::vector<int> splice_parts(Module& parent, const std::string& seg, const Parts& parts) {
    Graph& g = *parent.forward;
    int call = -1;
    for (auto& n : g.nodes)
        if (n.kind == NK::CallModule && n.target == seg) {
            if (call >= 0) throw Error("module '" + seg + "' is called more than once; cannot partition");
            call = n.id;
        }
    if (call < 0) throw Error("no call to '" + seg + "' found in parent graph");
    const Node call_node = g.at(call);

    Graph ng;
    ng.inputs = g.inputs;
    int next = g.max_id() + 1;
    std::vector<int> part_calls;
    std::unordered_map<int, int> alias;
    std::unordered_map<std::string, int> holder;  // boundary name -> node id in the parent
    for (auto& n : g.nodes) {
        if (n.id != call) {
            Node c = n;
            for (auto& a : c.args) {
                auto it = alias.find(a);
                if (it != alias.end()) a = it->second;
            }
            ng.nodes.push_back(std::move(c));
            continue;
        }
        for (size_t i = 0; i < parts.module_inputs.size(); ++i) holder[parts.module_inputs[i]] = call_node.args[i];
        for (size_t s = 0; s < parts.mods.size(); ++s) {
            Node pc;
            pc.id = next++;
            pc.kind = NK::CallModule;
            pc.target = seg + "_p" + std::to_string(s);
            for (auto& nm : parts.in_names[s]) pc.args.push_back(holder.at(nm));
            const int pid = pc.id;
            ng.nodes.push_back(std::move(pc));
            part_calls.push_back(pid);
            if (parts.out_names[s].size() == 1) {
                holder[parts.out_names[s][0]] = pid;
            } else {
                for (size_t k = 0; k < parts.out_names[s].size(); ++k) {
                    Node gi;
                    gi.id = next++;
                    gi.kind = NK::GetItem;
                    gi.args = {pid};
                    gi.attrs["index"] = (i64)k;
                    holder[parts.out_names[s][k]] = gi.id;
                    ng.nodes.push_back(std::move(gi));
                }
            }
        }
        alias[call] = parts.module_results.size() == 1 ? holder.at(parts.module_results[0]) : -1;
    }
    if (parts.module_results.size() > 1) {  // the parent read the results through get_item nodes
        Graph fixed;
        fixed.inputs = ng.inputs;
        std::unordered_map<int, int> item;
        for (auto& n : ng.nodes) {
            if (n.kind == NK::GetItem && !n.args.empty() && n.args[0] == -1) {
                item[n.id] = holder.at(parts.module_results.at((size_t)get_int(n.attrs, "index").value_or(0)));
                continue;
            }
            Node c = n;
            for (auto& a : c.args) {
                auto it = item.find(a);
                if (it != item.end()) a = it->second;
                if (a == -1) throw Error("partitioned multi-result module used without get_item");
            }
            fixed.nodes.push_back(std::move(c));
        }
        ng = std::move(fixed);
    } else {
        for (auto& n : ng.nodes)
            for (auto& a : n.args) {
                auto it = alias.find(a);
                if (it != alias.end()) a = it->second;
            }
    }
    ng.out = ng.nodes.back().id;
    ng.validate();
    parent.forward = std::move(ng);
    for (auto it = parent.children.begin(); it != parent.children.end(); ++it)
        if (it->name == seg) {
            parent.children.erase(it);
            break;
        }
    for (size_t s = 0; s < parts.mods.size(); ++s) parent.add_child(seg + "_p" + std::to_string(s), parts.mods[s]);
    part_calls.pop_back();
    return part_calls;
}

int depth_of(const std::string& p) { return p.empty() ? 0 : (int)std::count(p.begin(), p.end(), '.') + 1; }

}  // namespace

StagePlan build_stage_plan(const Module& model, const std::vector<SplitAnnotation>& splits) {
    if (splits.empty()) throw Error("no pipeline_split annotations");
    Module work = model;
    std::map<std::string, std::vector<int>> cuts;  // site -> boundary call ids in its current graph
    for (auto& sp : splits) {
        const Module* site = work.resolve(sp.site);
        if (!site) throw Error("unknown module path '" + sp.site + "'");
        if (!site->forward) throw Error("pipeline_split target '" + sp.site + "' has no graph");
        int id = -1;
        for (auto& n : site->forward->nodes)
            if (n.kind == NK::CallModule && n.target == sp.after_child) id = n.id;
        if (id < 0)
            throw Error("pipeline boundary not found: no call to '" + sp.after_child + "' in '" + sp.site + "'");
        cuts[sp.site].push_back(id);
    }
    while (!(cuts.size() == 1 && cuts.begin()->first.empty())) {
        // deepest annotated site first; among equals the lexicographically smallest
        auto pick = cuts.begin();
        for (auto it = cuts.begin(); it != cuts.end(); ++it)
            if (depth_of(it->first) > depth_of(pick->first) ||
                (depth_of(it->first) == depth_of(pick->first) && it->first < pick->first))
                pick = it;
        const std::string site = pick->first;
        const std::vector<int> b = pick->second;
        cuts.erase(pick);

        Module* m = work.resolve(site);
        Parts parts = cut_module(*m, b, module_input_specs_at(work, site));
        const std::string parent = parent_of(site), seg = last_of(site);
        Module* pm = work.resolve(parent);
        if (!pm || !pm->forward) throw Error("cannot propagate pipeline annotations into '" + parent + "'");
        int replaced = -1;
        for (auto& n : pm->forward->nodes)
            if (n.kind == NK::CallModule && n.target == seg) replaced = n.id;
        std::vector<int> nb = splice_parts(*pm, seg, parts);
        int last_call = -1;
        for (auto& n : pm->forward->nodes)
            if (n.kind == NK::CallModule && n.target == seg + "_p" + std::to_string(parts.mods.size() - 1))
                last_call = n.id;
        auto& pc = cuts[parent];
        for (auto& x : pc)
            if (x == replaced) x = last_call;
        pc.insert(pc.end(), nb.begin(), nb.end());
    }
    Parts top = cut_module(work, cuts[""], declared_inputs(*work.forward));
    StagePlan plan;
    plan.model_inputs = top.module_inputs;
    plan.model_outputs = top.module_results;
    for (size_t s = 0; s < top.mods.size(); ++s) {
        Stage st;
        st.module = std::move(top.mods[s]);
        st.module.name = "stage" + std::to_string(s);
        st.consumes = top.in_names[s];
        st.produces = top.out_names[s];
        plan.stages.push_back(std::move(st));
    }
    return plan;
}

}  // namespace sb
