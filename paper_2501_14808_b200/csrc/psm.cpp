// psm.cpp -- Prefix Sharing Maximization (HyGen §4.3; Alg. 3,
// P:534-583): offline requests live in a prefix tree T_p
// over their prompt tokens; the offline phase admits them in the tree's DFS
// order, so requests that share a prefix land in the same batch and their
// prefix KV can be shared (the prefix-group pass of hg_hybrid_attention).
//
// DFS order: at a node, the requests whose prompt ends there (insertion order),
// then the children in order of first insertion into the live tree.  The DFS
// list is rebuilt (O(live nodes)) only after inserts, as the paper's
// "pre-processed list ... synced up with the prefix tree": a removal
// marks its list entry dead (O(1)) and prunes the subtree it emptied, and
// readers skip dead entries from a cursor -- so Alg. 3's "take the next DFS
// request, remove it" loop costs O(1) amortised per admitted request.  The
// LCP of two live entries separated by dead ones is the minimum of the
// adjacent LCPs between them (trie preorder).
#include <algorithm>
#include <climits>
#include <unordered_map>
#include <vector>

#include "hg_internal.h"

using namespace hg;

struct hg_psm {
    struct Node {
        std::vector<std::pair<int32_t, int32_t>> kids;  // (token, node) in first-insertion order
        std::unordered_map<int32_t, int32_t> index;     // token -> node
        std::vector<int32_t> reqs;                       // requests ending here
        int32_t depth = 0, parent = -1, token = 0;
    };
    std::vector<Node> nodes{1};
    std::vector<int32_t> free_nodes;                     // pruned node slots for reuse
    std::unordered_map<int32_t, int32_t> where;          // request -> node
    std::unordered_map<int32_t, int32_t> pos;            // request -> index in `order` (valid when !dirty)
    std::vector<int32_t> order;                          // DFS list of requests
    std::vector<int32_t> lcp;                            // LCP with the DFS predecessor in `order`
    std::vector<char> dead;                              // removed since the last rebuild
    size_t head = 0;                                     // first possibly-live entry of `order`
    bool dirty = false;
    int32_t live = 0;

    int32_t new_node(int32_t parent, int32_t token) {
        int32_t id;
        if (!free_nodes.empty()) {
            id = free_nodes.back();
            free_nodes.pop_back();
            nodes[id] = Node();
        } else {
            id = (int32_t)nodes.size();
            nodes.emplace_back();
        }
        nodes[id].parent = parent;
        nodes[id].token = token;
        nodes[id].depth = nodes[parent].depth + 1;
        return id;
    }
    // drop empty leaves upward from `n` (never the root)
    void prune(int32_t n) {
        while (n != 0 && nodes[n].reqs.empty() && nodes[n].kids.empty()) {
            Node &par = nodes[nodes[n].parent];
            par.index.erase(nodes[n].token);
            par.kids.erase(std::find(par.kids.begin(), par.kids.end(), std::make_pair(nodes[n].token, n)));
            const int32_t up = nodes[n].parent;
            nodes[n] = Node();
            free_nodes.push_back(n);
            n = up;
        }
    }
    void rebuild() {
        order.clear();
        lcp.clear();
        pos.clear();
        // iterative preorder; track, for every emitted request, the depth of the
        // deepest common ancestor with the previously emitted request
        struct Frame { int32_t node, next_kid; };
        std::vector<Frame> st{{0, 0}};
        int32_t min_depth_since = 0;  // shallowest node on the path walked since the last emitted request
        bool first = true;
        bool enter = true;
        while (!st.empty()) {
            Frame &f = st.back();
            Node &n = nodes[f.node];
            if (enter) {
                for (int32_t r : n.reqs) {
                    pos[r] = (int32_t)order.size();
                    order.push_back(r);
                    lcp.push_back(first ? 0 : min_depth_since);
                    first = false;
                    min_depth_since = n.depth;
                }
            }
            if (f.next_kid < (int32_t)n.kids.size()) {
                const int32_t child = n.kids[f.next_kid++].second;
                st.push_back({child, 0});
                enter = true;
            } else {
                st.pop_back();
                enter = false;
                if (!st.empty()) min_depth_since = std::min(min_depth_since, nodes[st.back().node].depth);
            }
        }
        dead.assign(order.size(), 0);
        head = 0;
        dirty = false;
    }
};

extern "C" hg_status hg_psm_create(hg_psm **out) {
    if (!out) return fail(HG_E_INVALID, "NULL argument");
    *out = new hg_psm();
    return HG_OK;
}

extern "C" hg_status hg_psm_destroy(hg_psm *p) {
    delete p;
    return HG_OK;
}

extern "C" hg_status hg_psm_insert(hg_psm *p, int32_t rid, const int32_t *tokens, int32_t n) {
    if (!p || n < 0 || (n > 0 && !tokens)) return fail(HG_E_INVALID, "bad arguments");
    if (p->where.count(rid)) return fail(HG_E_INVALID, "request %d already in the prefix tree", rid);
    int32_t cur = 0;
    for (int32_t k = 0; k < n; ++k) {
        auto it = p->nodes[cur].index.find(tokens[k]);
        if (it == p->nodes[cur].index.end()) {
            const int32_t nn = p->new_node(cur, tokens[k]);
            p->nodes[cur].index.emplace(tokens[k], nn);
            p->nodes[cur].kids.push_back({tokens[k], nn});
            cur = nn;
        } else {
            cur = it->second;
        }
    }
    p->nodes[cur].reqs.push_back(rid);
    p->where[rid] = cur;
    p->live++;
    p->dirty = true;
    return HG_OK;
}

extern "C" hg_status hg_psm_remove(hg_psm *p, int32_t rid) {
    if (!p) return fail(HG_E_INVALID, "NULL argument");
    auto it = p->where.find(rid);
    if (it == p->where.end()) return fail(HG_E_INVALID, "request %d not in the prefix tree", rid);
    const int32_t node = it->second;
    auto &v = p->nodes[node].reqs;
    v.erase(std::find(v.begin(), v.end(), rid));
    p->where.erase(it);
    if (!p->dirty) p->dead[p->pos[rid]] = 1;   // the DFS list stays valid: skip the entry
    p->prune(node);
    p->live--;
    return HG_OK;
}

extern "C" int32_t hg_psm_size(const hg_psm *p) { return p ? p->live : 0; }

extern "C" hg_status hg_psm_dfs_order(hg_psm *p, int32_t *ids, int32_t *lcp, int32_t max, int32_t *n_out) {
    if (!p || !n_out || max < 0 || (max > 0 && !ids)) return fail(HG_E_INVALID, "bad arguments");
    if (p->dirty) p->rebuild();
    while (p->head < p->order.size() && p->dead[p->head]) ++p->head;
    int32_t n = 0;
    int32_t run_min = 0;   // min adjacent LCP since the last emitted live entry
    for (size_t k = p->head; k < p->order.size() && n < max; ++k) {
        run_min = (n == 0) ? 0 : std::min(run_min, p->lcp[k]);
        if (p->dead[k]) continue;
        ids[n] = p->order[k];
        if (lcp) lcp[n] = run_min;
        ++n;
        run_min = INT32_MAX;
    }
    *n_out = n;
    return HG_OK;
}
