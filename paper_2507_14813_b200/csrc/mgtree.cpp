// mgtree.cpp -- MG-Tree compiler (step a1).
//
// Algorithm 2 "MG-Tree Construction" groups motifs by their edge
// at temporal rank T, recursing on T+1; node reuse for undivided groups and the
// |E(M)| = T check make each MG-Tree node a distinct edge prefix C_N shared by its
// descendants (definition).  Reading R8: the
// MG-Tree is the path-compressed trie of CANONICAL edge sequences.  We compile
//   (1) the full trie -- one row per distinct canonical prefix -- into the kernel
//       table (each row = one motif edge to match, Algo 3's per-edge step), and
//   (2) the path-compressed view (root, branching prefixes, query motifs) for the
//       Similarity Metric and the Fig. 6-style dump.
// Per row the compiler precomputes what Algorithm 1 decides at run time
// (PAPER.md:205-222): the candidate source ("anchor"), the structural check and
// which motif vertices become mapped -- the paper's "register-bound context
// mapping" / "predicated control flow" specialisation (§5.1.2)
// expressed as table data.
#include <algorithm>
#include <cstdio>
#include <map>

#include "internal.h"

namespace mayura {
namespace {

struct TrieNode {
    int parent = -1;
    uint8_t u = 0, v = 1;
    int depth = 1;    // edges in the prefix
    uint8_t nv = 2;   // distinct motif vertices in the prefix (canonical: labels 0..nv-1)
    std::vector<int> children;
    std::vector<uint32_t> motifs;  // input motifs equal to this prefix (Q_N)
};

typedef std::vector<std::pair<uint32_t, uint32_t>> Edges;

// First-appearance relabelling, u before v (reading R7).
Edges canonicalize(const Edges &m) {
    std::map<uint32_t, uint32_t> lab;
    Edges out;
    for (auto &e : m) {
        for (uint32_t x : {e.first, e.second})
            if (!lab.count(x)) {
                uint32_t id = (uint32_t)lab.size();
                lab[x] = id;
            }
        out.push_back({lab[e.first], lab[e.second]});
    }
    return out;
}

uint32_t n_vertices_of(const Edges &m) {
    uint32_t n = 0;
    for (auto &e : m) n = std::max(n, std::max(e.first, e.second) + 1);
    return n;
}

std::vector<TrieNode> build_trie(const std::vector<Edges> &motifs, const std::vector<uint32_t> &ids) {
    std::vector<TrieNode> trie(1);  // root = canonical first edge 0->1
    for (size_t k = 0; k < motifs.size(); k++) {
        const Edges &m = motifs[k];
        int cur = 0;
        for (size_t j = 1; j < m.size(); j++) {
            int nxt = -1;
            for (int c : trie[cur].children)
                if (trie[c].u == m[j].first && trie[c].v == m[j].second) nxt = c;
            if (nxt < 0) {
                TrieNode n;
                n.parent = cur;
                n.u = (uint8_t)m[j].first;
                n.v = (uint8_t)m[j].second;
                n.depth = trie[cur].depth + 1;
                n.nv = (uint8_t)std::max<uint32_t>(trie[cur].nv, std::max(m[j].first, m[j].second) + 1);
                nxt = (int)trie.size();
                trie.push_back(n);
                trie[cur].children.push_back(nxt);
            }
            cur = nxt;
        }
        trie[cur].motifs.push_back(ids[k]);
    }
    return trie;
}

// Flatten the trie to the kernel table (BFS, children contiguous and grouped by anchor).
mayura_status flatten(const std::vector<TrieNode> &trie, uint32_t n_motifs_total, Table &tab) {
    tab.nodes.clear();
    tab.groups.clear();
    tab.motif_node.assign(n_motifs_total, 0xFFFFFFFFu);
    std::vector<int> row_of(trie.size(), -1), trie_of;
    row_of[0] = 0;
    trie_of.push_back(0);
    DNode root{};
    root.want = CLS_NEW;
    root.n_new = 2;
    root.nv = 2;
    tab.nodes.push_back(root);
    for (size_t q = 0; q < trie_of.size(); q++) {
        const TrieNode &x = trie[trie_of[q]];
        DNode &dx = tab.nodes[q];
        dx.flags = (x.motifs.empty() ? 0 : NODE_COMPLETION) | (x.children.empty() ? 0 : NODE_INNER);
        for (uint32_t mi : x.motifs) tab.motif_node[mi] = (uint32_t)q;
        // group children by anchor (first-appearance order)
        std::vector<std::pair<std::pair<int, int>, std::vector<int>>> groups;
        for (int c : x.children) {
            const TrieNode &tc = trie[c];
            int kind, anchor;
            if (tc.u < x.nv) {
                kind = ANCHOR_OUT;
                anchor = tc.u;
            } else if (tc.v < x.nv) {
                kind = ANCHOR_IN;
                anchor = tc.v;
            } else {
                kind = ANCHOR_GLOBAL;
                anchor = 0;
            }
            auto key = std::make_pair(kind, anchor);
            auto it = std::find_if(groups.begin(), groups.end(),
                                   [&](const std::pair<std::pair<int, int>, std::vector<int>> &g) { return g.first == key; });
            if (it == groups.end()) groups.push_back({key, {c}});
            else it->second.push_back(c);
        }
        uint32_t gb = (uint32_t)tab.groups.size();
        for (auto &g : groups) {
            DGroup dg{};
            dg.kind = (uint8_t)g.first.first;
            dg.anchor = (uint8_t)g.first.second;
            // window start source: the node's own edge (x.u -> x.v) gives exact successor
            // pointers for its endpoints; the root edge (0 -> 1) a lower bound for 0 and 1.
            if (dg.kind == ANCHOR_GLOBAL) dg.start = START_GLOBAL;
            else if (dg.kind == ANCHOR_OUT)
                dg.start = dg.anchor == x.u ? START_P0 : dg.anchor == x.v ? START_P2
                         : dg.anchor == 0 ? START_R0 : dg.anchor == 1 ? START_R2 : START_SEARCH;
            else
                dg.start = dg.anchor == x.v ? START_P1 : dg.anchor == x.u ? START_P3
                         : dg.anchor == 1 ? START_R1 : dg.anchor == 0 ? START_R3 : START_SEARCH;
            dg.child_begin = (uint16_t)trie_of.size();
            uint32_t inner = 0;
            for (int c : g.second) {
                const TrieNode &tc = trie[c];
                DNode dn{};
                if (dg.kind == ANCHOR_OUT) {
                    dn.want = tc.v < x.nv ? tc.v : CLS_NEW;
                    dn.n_new = tc.v < x.nv ? 0 : 1;
                } else {
                    dn.want = CLS_NEW;
                    dn.n_new = dg.kind == ANCHOR_IN ? 1 : 2;
                }
                dn.nv = tc.nv;
                if (!tc.children.empty()) inner++;
                row_of[c] = (int)trie_of.size();
                trie_of.push_back(c);
                tab.nodes.push_back(dn);
            }
            dg.child_end = (uint16_t)trie_of.size();
            dg.n_inner = (uint8_t)inner;
            tab.groups.push_back(dg);
            if (trie_of.size() > MAYURA_MAX_TRIE_NODES)
                return fail(MAYURA_E_LIMIT, "mayura_build_mgtree: more than MAYURA_MAX_TRIE_NODES prefixes");
        }
        // dx may be invalidated by push_back: re-index
        tab.nodes[q].group_begin = (uint16_t)gb;
        tab.nodes[q].group_end = (uint16_t)tab.groups.size();
        bool sweep = !x.children.empty();
        for (uint32_t gi = gb; gi < tab.groups.size(); gi++) {
            const DGroup &dg = tab.groups[gi];
            sweep = sweep && dg.kind != ANCHOR_GLOBAL && dg.start < START_SEARCH && dg.n_inner == 0 &&
                    (uint32_t)(dg.child_end - dg.child_begin) <= kSweepChildren;
        }
        if (sweep) tab.nodes[q].flags |= NODE_SWEEP;
    }
    return MAYURA_OK;
}

// Path-compressed MG-Tree view: nodes = deepest prefix common to all motifs (root),
// branching prefixes and query-motif prefixes.  SM per PAPER.md:954-961.
void compressed_view(const std::vector<TrieNode> &trie, const std::vector<Edges> &canon,
                     uint32_t &n_nodes, double &sm, std::string &dump) {
    auto kept = [&](int i) { return trie[i].children.size() != 1 || !trie[i].motifs.empty(); };
    // root: walk down from trie row 0 while the node is a non-branching non-completion
    int root = 0;
    while (!kept(root)) root = trie[root].children[0];
    n_nodes = 0;
    double num = 0, den = 0;
    for (auto &m : canon) den += (double)m.size();
    dump.clear();
    // DFS over kept nodes
    std::vector<std::pair<int, std::pair<int, int>>> st;  // (trie node, (parent depth, indent))
    st.push_back({root, {0, 0}});
    while (!st.empty()) {
        int x = st.back().first;
        int pdepth = st.back().second.first, indent = st.back().second.second;
        st.pop_back();
        n_nodes++;
        num += trie[x].depth - pdepth;
        // reconstruct prefix edges
        std::vector<std::pair<int, int>> edges;
        for (int y = x; y >= 0; y = trie[y].parent) edges.push_back({trie[y].u, trie[y].v});
        std::reverse(edges.begin(), edges.end());
        std::string line(2 * indent, ' ');
        if (trie[x].motifs.empty()) line += "I";
        else {
            line += "Q=";
            for (size_t i = 0; i < trie[x].motifs.size(); i++)
                line += (i ? "," : "") + std::to_string(trie[x].motifs[i]);
        }
        line += " C=(";
        for (size_t i = 0; i < edges.size(); i++) {
            char b[32];
            snprintf(b, sizeof b, "%s%d>%d", i ? "," : "", edges[i].first, edges[i].second);
            line += b;
        }
        line += ")\n";
        dump += line;
        // children in the compressed tree: nearest kept descendants along each branch
        std::vector<int> kids;
        for (int c : trie[x].children) {
            int y = c;
            while (!kept(y)) y = trie[y].children[0];
            kids.push_back(y);
        }
        for (auto it = kids.rbegin(); it != kids.rend(); ++it) st.push_back({*it, {trie[x].depth, indent + 1}});
    }
    sm = den > 0 ? 1.0 - num / den : 0.0;
}

}  // namespace

mayura_status compile_tree(const uint32_t *motif_edges, const uint32_t *motif_len, uint32_t n_motifs,
                           int64_t delta, mayura_mgtree_s *m) {
    if (!motif_edges || !motif_len || n_motifs == 0)
        return fail(MAYURA_E_INVALID, "mayura_build_mgtree: empty group or NULL pointer");
    if (delta < 0) return fail(MAYURA_E_INVALID, "mayura_build_mgtree: delta < 0");
    if (n_motifs > MAYURA_MAX_MOTIFS) return fail(MAYURA_E_LIMIT, "mayura_build_mgtree: too many motifs");
    m->delta = delta;
    m->n_motifs = n_motifs;
    m->canon.clear();
    uint64_t off = 0;
    uint32_t maxv = 0, maxe = 0;
    for (uint32_t i = 0; i < n_motifs; i++) {
        uint32_t len = motif_len[i];
        if (len == 0 || len > MAYURA_MAX_EDGES)
            return fail(MAYURA_E_LIMIT, "mayura_build_mgtree: motif " + std::to_string(i) +
                                            " has 0 or more than MAYURA_MAX_EDGES edges");
        Edges e;
        for (uint32_t j = 0; j < len; j++) {
            uint32_t u = motif_edges[2 * (off + j)], v = motif_edges[2 * (off + j) + 1];
            if (u == v)
                return fail(MAYURA_E_INVALID, "mayura_build_mgtree: motif " + std::to_string(i) + " has a self-loop edge");
            e.push_back({u, v});
        }
        off += len;
        Edges c = canonicalize(e);
        uint32_t nv = n_vertices_of(c);
        if (nv > MAYURA_MAX_V)
            return fail(MAYURA_E_LIMIT, "mayura_build_mgtree: motif " + std::to_string(i) + " has more than MAYURA_MAX_V vertices");
        maxv = std::max(maxv, nv);
        maxe = std::max(maxe, len);
        m->canon.push_back(c);
    }
    std::vector<uint32_t> ids(n_motifs);
    for (uint32_t i = 0; i < n_motifs; i++) ids[i] = i;
    std::vector<TrieNode> trie = build_trie(m->canon, ids);
    mayura_status s = flatten(trie, n_motifs, m->group);
    if (s != MAYURA_OK) return s;
    m->group.max_vertices = maxv;
    m->group.max_edges = maxe;
    compressed_view(trie, m->canon, m->n_mg_nodes, m->sm, m->dump);
    m->single.assign(n_motifs, Table());
    for (uint32_t i = 0; i < n_motifs; i++) {
        std::vector<Edges> one{m->canon[i]};
        std::vector<uint32_t> id0{0};
        std::vector<TrieNode> t1 = build_trie(one, id0);
        s = flatten(t1, 1, m->single[i]);
        if (s != MAYURA_OK) return s;
        m->single[i].max_vertices = n_vertices_of(m->canon[i]);
        m->single[i].max_edges = (uint32_t)m->canon[i].size();
    }
    return MAYURA_OK;
}

}  // namespace mayura
