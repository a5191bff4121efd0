// bsim_host.cu -- the pipelined host-buffer control step (bsim_env_step_host):
// EnvBatch.step called with host arrays (reference envs.py:178-200, whose
// numpy step returns host obs / reward / done) as ONE native call, so the
// per-step host work is a single ctypes crossing instead of a dozen
// Python-side copies, stream switches and event records.
//
// Schedule for n chunks of envs (one per step-kernel wave by default):
//   copy stream:    H2D a_0 .. a_{n-1} | wait done_0, D2H out_0 | wait done_1, D2H out_1 ...
//   chunk stream c: wait in_c, step range c (physics + task tail), record done_c
// Chunk c > 0 launches on its own stream, so its CTAs take the SMs as chunk
// c-1's retire (the wave tail of one launch, not of n serialised launches),
// and chunk c's outputs cross PCIe while later chunks still step.
#include <cuda_runtime.h>

#include <string>
#include <vector>

#include "batchsim_b200.h"

namespace {

constexpr int MAX_CHUNKS = 16;

struct Pool {   // per-device streams / events, created on first use
    int dev = -1;
    cudaStream_t copy = nullptr;
    cudaStream_t comp[MAX_CHUNKS] = {};
    cudaEvent_t start = nullptr, in[MAX_CHUNKS] = {}, done[MAX_CHUNKS] = {}, end = nullptr;
};
std::vector<Pool> g_pools;
std::string h_err;

int fail(const char *what, cudaError_t e) {
    h_err = std::string(what) + ": " + cudaGetErrorString(e);
    return BSIM_E_CUDA;
}

int pool_for_device(Pool **out) {
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return fail("cudaGetDevice", e);
    for (auto &p : g_pools)
        if (p.dev == dev) {
            *out = &p;
            return BSIM_OK;
        }
    Pool p;
    p.dev = dev;
    const unsigned ev_flags = cudaEventDisableTiming;
    if ((e = cudaStreamCreateWithFlags(&p.copy, cudaStreamNonBlocking)) != cudaSuccess) return fail("stream", e);
    for (int c = 0; c < MAX_CHUNKS; ++c) {
        if ((e = cudaStreamCreateWithFlags(&p.comp[c], cudaStreamNonBlocking)) != cudaSuccess) return fail("stream", e);
        if ((e = cudaEventCreateWithFlags(&p.in[c], ev_flags)) != cudaSuccess) return fail("event", e);
        if ((e = cudaEventCreateWithFlags(&p.done[c], ev_flags)) != cudaSuccess) return fail("event", e);
    }
    if ((e = cudaEventCreateWithFlags(&p.start, ev_flags)) != cudaSuccess) return fail("event", e);
    if ((e = cudaEventCreateWithFlags(&p.end, ev_flags)) != cudaSuccess) return fail("event", e);
    g_pools.push_back(p);
    *out = &g_pools.back();
    return BSIM_OK;
}

template <class R> struct Api;
template <> struct Api<float> {
    using P = bsim_params_t;
    using S = bsim_state_t;
    static int step(const bsim_layout_t *l, const P *p, const S *s, int32_t n, const bsim_actions_t *a, int32_t b,
                    int32_t c, void *st) { return bsim_step_range(l, p, s, n, a, b, c, st); }
    static int env_step(const bsim_layout_t *l, const P *p, const S *s, int32_t n, const bsim_actions_t *a,
                        const bsim_task_t *t, int32_t b, int32_t c, void *st) {
        return bsim_env_step_range(l, p, s, n, a, t, b, c, st);
    }
    static int task(const bsim_layout_t *l, const S *s, const bsim_task_t *t, int32_t b, int32_t c, void *st) {
        return bsim_task_step_range(l, s, t, b, c, st);
    }
};
template <> struct Api<double> {
    using P = bsim_params64_t;
    using S = bsim_state64_t;
    static int step(const bsim_layout_t *l, const P *p, const S *s, int32_t n, const bsim_actions_t *a, int32_t b,
                    int32_t c, void *st) { return bsim_step_range_f64(l, p, s, n, a, b, c, st); }
    static int env_step(const bsim_layout_t *l, const P *p, const S *s, int32_t n, const bsim_actions_t *a,
                        const bsim_task_t *t, int32_t b, int32_t c, void *st) {
        return bsim_env_step_range_f64(l, p, s, n, a, t, b, c, st);
    }
    static int task(const bsim_layout_t *l, const S *s, const bsim_task_t *t, int32_t b, int32_t c, void *st) {
        return bsim_task_step_range_f64(l, s, t, b, c, st);
    }
};

template <class R>
int step_host(const bsim_layout_t *l, const typename Api<R>::P *p, const typename Api<R>::S *s, int32_t n_sub,
              const bsim_actions_t *act, const bsim_task_t *t, const bsim_host_io_t *io, void *stream) {
    if (!l || !p || !s || !act || !act->actions || !t || !io || !io->actions || !io->obs || !io->reward ||
        !io->done || !io->timeout || !io->poisoned || t->act_dim != l->dofs_per_env) {
        h_err = "bsim_env_step_host: invalid arguments";
        return BSIM_E_INVALID;
    }
    const int E = l->num_envs;
    if (E == 0) return BSIM_OK;
    if (io->fused == 2) {   // zero-copy: one launch reading / writing the mapped host buffers
        cudaStream_t main = (cudaStream_t)stream;
        void *dp[6];
        const void *hp[6] = {io->actions, io->obs, io->reward, io->done, io->timeout, io->poisoned};
        for (int i = 0; i < 6; ++i) {
            cudaPointerAttributes at;
            cudaError_t e = cudaPointerGetAttributes(&at, hp[i]);
            if (e != cudaSuccess || at.type != cudaMemoryTypeHost || !at.devicePointer) {
                cudaGetLastError();
                h_err = "bsim_env_step_host: zero-copy mode needs page-locked (mapped) host buffers";
                return BSIM_E_INVALID;
            }
            dp[i] = at.devicePointer;
        }
        bsim_actions_t a2 = *act;
        a2.actions = dp[0];
        bsim_task_t t2 = *t;
        t2.obs = dp[1];
        t2.reward = dp[2];
        t2.done = (uint8_t *)dp[3];
        t2.timeout = (uint8_t *)dp[4];
        t2.poisoned = (uint8_t *)dp[5];
        int rc = Api<R>::env_step(l, p, s, n_sub, &a2, &t2, 0, E, main);
        if (rc != BSIM_OK) h_err = "bsim_env_step_host: zero-copy launch failed (see bsim_last_error)";
        return rc;
    }
    int n = io->n_chunks;
    if (n <= 0) {
        int32_t wave = 0;
        if (int rc = bsim_step_envs_per_wave(l, sizeof(R) == 8, &wave)) {
            h_err = "bsim_env_step_host: bsim_step_envs_per_wave failed";
            return rc;
        }
        n = wave > 0 ? (E + wave - 1) / wave : 1;
    }
    n = n < 1 ? 1 : (n > MAX_CHUNKS ? MAX_CHUNKS : (n > E ? E : n));
    Pool *pl = nullptr;
    if (int rc = pool_for_device(&pl)) return rc;
    cudaStream_t main = (cudaStream_t)stream, copy = pl->copy;
    cudaError_t e;
    // everything below runs after the work already queued on `stream`
    if ((e = cudaEventRecord(pl->start, main)) != cudaSuccess) return fail("cudaEventRecord", e);
    if ((e = cudaStreamWaitEvent(copy, pl->start, 0)) != cudaSuccess) return fail("cudaStreamWaitEvent", e);
    const size_t rs = sizeof(R), A = (size_t)t->act_dim, O = (size_t)t->obs_dim;
    auto lo = [&](int c) { return (int)((long)E * c / n); };
    for (int c = 0; c < n; ++c) {   // uploads first: chunk c+1's actions land while chunk c steps
        const size_t b = lo(c), m = lo(c + 1) - lo(c);
        e = cudaMemcpyAsync((char *)act->actions + b * A * rs, (const char *)io->actions + b * A * rs, m * A * rs,
                            cudaMemcpyHostToDevice, copy);
        if (e != cudaSuccess) return fail("cudaMemcpyAsync(actions)", e);
        if ((e = cudaEventRecord(pl->in[c], copy)) != cudaSuccess) return fail("cudaEventRecord", e);
    }
    for (int c = 0; c < n; ++c) {
        const int b = lo(c), m = lo(c + 1) - lo(c);
        cudaStream_t cs = pl->comp[c];
        if ((e = cudaStreamWaitEvent(cs, pl->start, 0)) != cudaSuccess) return fail("cudaStreamWaitEvent", e);
        if ((e = cudaStreamWaitEvent(cs, pl->in[c], 0)) != cudaSuccess) return fail("cudaStreamWaitEvent", e);
        int rc = io->fused ? Api<R>::env_step(l, p, s, n_sub, act, t, b, m, cs)
                           : Api<R>::step(l, p, s, n_sub, act, b, m, cs);
        if (rc == BSIM_OK && !io->fused) rc = Api<R>::task(l, s, t, b, m, cs);
        if (rc != BSIM_OK) {
            h_err = "bsim_env_step_host: chunk launch failed (see bsim_last_error / bsim_task_last_error)";
            return rc;
        }
        if ((e = cudaEventRecord(pl->done[c], cs)) != cudaSuccess) return fail("cudaEventRecord", e);
        if ((e = cudaStreamWaitEvent(copy, pl->done[c], 0)) != cudaSuccess) return fail("cudaStreamWaitEvent", e);
        struct {
            void *dst;
            const void *src;
            size_t bytes;
        } outs[5] = {
            {(char *)io->obs + b * O * rs, (const char *)t->obs + b * O * rs, m * O * rs},
            {(char *)io->reward + b * rs, (const char *)t->reward + b * rs, m * rs},
            {io->done + b, t->done + b, (size_t)m},
            {io->timeout + b, t->timeout + b, (size_t)m},
            {io->poisoned + b, t->poisoned + b, (size_t)m},
        };
        for (auto &o : outs)
            if ((e = cudaMemcpyAsync(o.dst, o.src, o.bytes, cudaMemcpyDeviceToHost, copy)) != cudaSuccess)
                return fail("cudaMemcpyAsync(outputs)", e);
    }
    // `stream` resumes after every chunk and every copy
    if ((e = cudaEventRecord(pl->end, copy)) != cudaSuccess) return fail("cudaEventRecord", e);
    if ((e = cudaStreamWaitEvent(main, pl->end, 0)) != cudaSuccess) return fail("cudaStreamWaitEvent", e);
    return BSIM_OK;
}

}  // namespace

// A captured host step: the whole schedule above as one CUDA graph (one
// cudaGraphLaunch per control step instead of ~20 API calls), plus an 8-byte
// upload of the post-step count into task->step_count_dev so the DR interval
// keeps advancing.  The action-upload nodes are re-pointed when the caller
// passes a different host array.
struct bsim_host_graph {
    cudaGraph_t graph = nullptr;
    cudaGraphExec_t exec = nullptr;
    const char *src = nullptr;            // host actions the upload nodes read
    std::vector<cudaGraphNode_t> up;      // the action-upload nodes
    std::vector<size_t> off, bytes;       // their source offsets / sizes
    std::vector<void *> dst;
    int64_t *count_host = nullptr;        // pinned slot the count upload reads
};

namespace {
template <class R>
int host_graph_create(const bsim_layout_t *l, const typename Api<R>::P *p, const typename Api<R>::S *s,
                      int32_t n_sub, const bsim_actions_t *act, const bsim_task_t *t, const bsim_host_io_t *io,
                      int64_t *count_host, bsim_host_graph **out) {
    if (!out || !t || !t->step_count_dev || !count_host || !io || !io->actions || !act || !act->actions ||
        io->fused == 2) {   // zero-copy is one launch with the host pointers baked in: nothing to capture
        h_err = "bsim_env_step_host_graph: invalid arguments";
        return BSIM_E_INVALID;
    }
    Pool *pl = nullptr;
    if (int rc = pool_for_device(&pl)) return rc;
    cudaStream_t cap;
    cudaError_t e = cudaStreamCreateWithFlags(&cap, cudaStreamNonBlocking);
    if (e != cudaSuccess) return fail("cudaStreamCreate", e);
    auto *g = new bsim_host_graph;
    g->count_host = count_host;
    g->src = (const char *)io->actions;
    int rc = BSIM_OK;
    if ((e = cudaStreamBeginCapture(cap, cudaStreamCaptureModeRelaxed)) != cudaSuccess) {
        rc = fail("cudaStreamBeginCapture", e);
    } else {
        e = cudaMemcpyAsync((void *)t->step_count_dev, count_host, sizeof(int64_t), cudaMemcpyHostToDevice, cap);
        rc = e != cudaSuccess ? fail("cudaMemcpyAsync(step count)", e) : step_host<R>(l, p, s, n_sub, act, t, io, cap);
        cudaError_t e2 = cudaStreamEndCapture(cap, &g->graph);
        if (rc == BSIM_OK && e2 != cudaSuccess) rc = fail("cudaStreamEndCapture", e2);
    }
    cudaStreamDestroy(cap);
    if (rc == BSIM_OK) {   // find the action uploads: host -> act->actions
        size_t n = 0;
        cudaGraphGetNodes(g->graph, nullptr, &n);
        std::vector<cudaGraphNode_t> nodes(n);
        cudaGraphGetNodes(g->graph, nodes.data(), &n);
        const size_t span = (size_t)l->num_envs * t->act_dim * sizeof(R);
        for (auto nd : nodes) {
            cudaGraphNodeType ty;
            cudaGraphNodeGetType(nd, &ty);
            if (ty != cudaGraphNodeTypeMemcpy) continue;
            cudaMemcpy3DParms mp;
            cudaGraphMemcpyNodeGetParams(nd, &mp);
            const char *sp = (const char *)mp.srcPtr.ptr, *dp = (const char *)mp.dstPtr.ptr;
            if (dp >= (const char *)act->actions && dp < (const char *)act->actions + span) {
                g->up.push_back(nd);
                g->off.push_back((size_t)(sp - g->src));
                g->bytes.push_back(mp.extent.width * mp.extent.height * mp.extent.depth);
                g->dst.push_back(mp.dstPtr.ptr);
            }
        }
        if ((e = cudaGraphInstantiate(&g->exec, g->graph, 0)) != cudaSuccess) rc = fail("cudaGraphInstantiate", e);
    }
    if (rc != BSIM_OK) {
        if (g->graph) cudaGraphDestroy(g->graph);
        delete g;
        return rc;
    }
    *out = g;
    return BSIM_OK;
}
}  // namespace

extern "C" {
int bsim_env_step_host_graph(const bsim_layout_t *l, const bsim_params_t *p, const bsim_state_t *s, int32_t n,
                             const bsim_actions_t *a, const bsim_task_t *t, const bsim_host_io_t *io,
                             int64_t *count_host, bsim_host_graph **out) {
    return host_graph_create<float>(l, p, s, n, a, t, io, count_host, out);
}
int bsim_env_step_host_graph_f64(const bsim_layout_t *l, const bsim_params64_t *p, const bsim_state64_t *s,
                                 int32_t n, const bsim_actions_t *a, const bsim_task_t *t,
                                 const bsim_host_io_t *io, int64_t *count_host, bsim_host_graph **out) {
    return host_graph_create<double>(l, p, s, n, a, t, io, count_host, out);
}
int bsim_host_graph_launch(bsim_host_graph *g, const void *host_actions, int64_t step_count, void *stream) {
    if (!g || !host_actions) {
        h_err = "bsim_host_graph_launch: invalid arguments";
        return BSIM_E_INVALID;
    }
    cudaError_t e;
    if ((const char *)host_actions != g->src) {
        for (size_t i = 0; i < g->up.size(); ++i) {
            e = cudaGraphExecMemcpyNodeSetParams1D(g->exec, g->up[i], g->dst[i],
                                                   (const char *)host_actions + g->off[i], g->bytes[i],
                                                   cudaMemcpyHostToDevice);
            if (e != cudaSuccess) return fail("cudaGraphExecMemcpyNodeSetParams1D", e);
        }
        g->src = (const char *)host_actions;
    }
    *g->count_host = step_count;   // the previous launch has retired (the caller synchronised)
    if ((e = cudaGraphLaunch(g->exec, (cudaStream_t)stream)) != cudaSuccess) return fail("cudaGraphLaunch", e);
    return BSIM_OK;
}
void bsim_host_graph_destroy(bsim_host_graph *g) {
    if (!g) return;
    if (g->exec) cudaGraphExecDestroy(g->exec);
    if (g->graph) cudaGraphDestroy(g->graph);
    delete g;
}

int bsim_env_step_host(const bsim_layout_t *l, const bsim_params_t *p, const bsim_state_t *s, int32_t n,
                       const bsim_actions_t *a, const bsim_task_t *t, const bsim_host_io_t *io, void *st) {
    return step_host<float>(l, p, s, n, a, t, io, st);
}
int bsim_env_step_host_f64(const bsim_layout_t *l, const bsim_params64_t *p, const bsim_state64_t *s, int32_t n,
                           const bsim_actions_t *a, const bsim_task_t *t, const bsim_host_io_t *io, void *st) {
    return step_host<double>(l, p, s, n, a, t, io, st);
}
const char *bsim_host_last_error(void) { return h_err.c_str(); }
}
