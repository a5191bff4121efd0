// TEST-ONLY host build of the step kernel's per-env body (bsim_step.cuh),
// so the CUDA code path's arithmetic can be debugged against the oracle on a
// CPU-only machine.  Mirrors step_kernel()'s load / stage / substep / store
// sequence in CTA-sized env groups (stride NE + 1).  Never used by the product.
#include <algorithm>
#include <cstdlib>
#include <vector>

#include "../../paper_2108_10470_b200/csrc/bsim_step.cuh"
#include "../../paper_2108_10470_b200/csrc/bsim_topologies.cuh"

using namespace bsim;

template <class R, class T>
static void run_t(const bsim_layout_t *L, const typename Abi<R>::Params *p, const typename Abi<R>::State *s,
                int n_substeps) {
    Ctx<R> c;
    c.L = *L;
    c.p = *p;
    c.s = *s;
    c.d = make_dims(*L, sizeof(R) == 8);
    c.joints = reinterpret_cast<const typename Abi<R>::Joint *>(L->joints);
    const Dims &d = c.d;
    // the batch in CTA-sized groups of Shape<R>::NE envs, one "thread" each
    constexpr int NE = Shape<R>::NE;
    const int E = d.E;
    std::vector<R> buf((size_t)d.pad * NE);
    for (int e0 = 0; e0 < E; e0 += NE) {
        const int ne = E - e0 < NE ? E - e0 : NE;
        std::fill(buf.begin(), buf.end(), R(1e30));   // poison: catches unstaged reads
        Grp<R> g{buf.data(), e0, ne, 0, 1, 0, d.pad,
                 JTab<R>{reinterpret_cast<const unsigned char *>(c.joints), (int)sizeof(*c.joints)}};
        for (int el = 0; el < ne; ++el)
            for (int b = 0; b < d.B; ++b)
                for (int k = 0; k < 13; ++k)
                    g.env(el).at(ib(d, b, body_item13(k))) = s->body_q[13 * ((size_t)(e0 + el) * d.B + b) + k];
        stage_group(c, g);
        for (int st = 0; st < n_substeps; ++st) {
            group_step<R, T>(c, g, st == n_substeps - 1, st);
            if (d.T && st != n_substeps - 1) readout_group(c, g);
        }
        readout_group(c, g);
        for (int el = 0; el < ne; ++el) {
            const int e = e0 + el;
            Ws<R> w = g.env(el);
            for (int i = 0; i < d.P; ++i)
                for (int k = 0; k < 3; ++k)
                    s->friction_anchor[3 * ((size_t)i * E + e) + k] = w.at(d.o_anchor + ANCHOR_ITEMS * i + k);
            for (int b = 0; b < d.B; ++b)
                for (int k = 0; k < 13; ++k) {
                    R x = w.at(ib(d, b, body_item13(k)));
                    s->body_q[13 * ((size_t)e * d.B + b) + k] = x;
                    s->body_state[13 * ((size_t)e * d.B + b) + k] = k < 3 ? x + s->env_origins[3 * e + k] : x;
                }
            for (int a = 0; a < d.A; ++a)
                for (int k = 0; k < 13; ++k)
                    s->root_state[13 * ((size_t)e * d.A + a) + k] =
                        s->body_state[13 * ((size_t)e * d.B + L->actor_body_offset[a]) + k];
        }
    }
}

template <class R>
static void run(const bsim_layout_t *L, const typename Abi<R>::Params *p, const typename Abi<R>::State *s, int n) {
    switch (L->topology_id) {
#define HK_TOPO(ID, TYPE) \
    case ID:              \
        return run_t<R, TYPE>(L, p, s, n);
        BSIM_TOPOLOGIES(HK_TOPO)
        BSIM_TOPOLOGIES_LARGE(HK_TOPO)
#undef HK_TOPO
    default:
        return run_t<R, TopoGeneric>(L, p, s, n);
    }
}

extern "C" void hk_step(const bsim_layout_t *L, const bsim_params_t *p, const bsim_state_t *s, int n) {
    run<float>(L, p, s, n);
}
extern "C" void hk_step_f64(const bsim_layout_t *L, const bsim_params64_t *p, const bsim_state64_t *s, int n) {
    run<double>(L, p, s, n);
}
