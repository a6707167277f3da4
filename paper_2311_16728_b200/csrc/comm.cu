// comm.cu -- A10 + A11 fused over peer memory (SURVEY §8(e) extension f3): one kernel that, on
// every rank, sums its shard of the gradient over all ranks, applies Adam to that shard and
// writes the updated parameters (and zeroed gradients) into every rank's buffers.
//
// The path is data parallel over keyframe views (north_star): each rank's backward adds its
// views' gradient into its own [K][ld] gradient buffer; the batch gradient is the sum over
// ranks (R22).  Instead of NCCL reduce-scatter -> Adam -> all-gather (three launches, the
// gradient and the parameters each crossing NVLink once, an intermediate shard in HBM), rank g
// owns the flat element range [e_g, e_{g+1}) of the [K][ld] buffer and
//   * reads the gradient of every rank for those elements -- with NVLink SHARP (NVLS) as one
//     multimem.ld_reduce on the multicast address (the switch adds), else peer loads summed in
//     rank order 0..G-1 -- so the reduced gradient never touches HBM;
//   * runs the Adam update of those elements (the arithmetic of gs_adam_step, adam1 in
//     gs_internal.cuh: the same bits) on its 1/G share of the moments;
//   * stores the new parameter value, and 0 into the gradient, to every rank -- one
//     multimem.st on the multicast address, else one peer store per rank.
// Two peer barriers (k_peer_barrier) bracket the kernel: before, every rank's backward is done;
// after, every rank's parameters are complete before the next projection reads them.  Every
// rank computes different elements and broadcasts them, so the replicas stay bit-identical.
//
// Buffers are symmetric (same size on every rank, mapped into every peer's address space by
// the caller -- torch symmetric memory); this file never allocates.
#include "gs_internal.cuh"

namespace gsk {

constexpr int COMM_MAX_WORLD = 8;
struct PeerPtrs {
    float *p[COMM_MAX_WORLD];
};
struct PeerFlags {
    uint32_t *p[COMM_MAX_WORLD];
};

__device__ __forceinline__ void st_release_sys(uint32_t *a, uint32_t v) {
    asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(a), "r"(v) : "memory");
}
__device__ __forceinline__ uint32_t ld_acquire_sys(const uint32_t *a) {
    uint32_t v;
    asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(a) : "memory");
    return v;
}

// One CTA of `world` threads.  flags.p[q] = rank q's flag array (uint32[world]); thread q
// announces epoch e to rank q (its slot `rank`), then waits until rank q has announced e here.
// epoch_dev: this rank's barrier count (device; every rank calls the barrier the same number
// of times, so counts agree without a host round trip -- a captured graph replays correctly).
// step_dev (optional): the Adam step counter, incremented once the barrier has passed.
__global__ void k_peer_barrier(PeerFlags flags, int rank, int world, uint32_t *epoch_dev, int64_t *step_dev) {
    const uint32_t e = *epoch_dev + 1u;
    const int q = threadIdx.x;
    __threadfence_system();  // this rank's earlier writes (its backward, its broadcasts) first
    if (q < world) {
        st_release_sys(flags.p[q] + rank, e);
        const uint32_t *mine = flags.p[rank] + q;
        while ((int32_t)(ld_acquire_sys(mine) - e) < 0) {
        }
    }
    __syncthreads();
    if (q == 0) {
        *epoch_dev = e;
        if (step_dev) *step_dev += 1;
    }
}

// peer loads / stores at system scope (the peers' buffers are other GPUs' memory over NVLink)
__device__ __forceinline__ float4 ld_sys(const float *addr) {
    float4 r;
    asm volatile("ld.relaxed.sys.global.v4.f32 {%0, %1, %2, %3}, [%4];"
                 : "=f"(r.x), "=f"(r.y), "=f"(r.z), "=f"(r.w)
                 : "l"(addr)
                 : "memory");
    return r;
}
__device__ __forceinline__ void st_sys(float *addr, float4 v) {
    asm volatile("st.relaxed.sys.global.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(addr), "f"(v.x), "f"(v.y), "f"(v.z),
                 "f"(v.w)
                 : "memory");
}

__device__ __forceinline__ float4 mc_ld_reduce(const float *addr) {
    float4 r;
    asm volatile("multimem.ld_reduce.relaxed.sys.global.add.v4.f32 {%0, %1, %2, %3}, [%4];"
                 : "=f"(r.x), "=f"(r.y), "=f"(r.z), "=f"(r.w)
                 : "l"(addr)
                 : "memory");
    return r;
}
__device__ __forceinline__ void mc_st(float *addr, float4 v) {
    asm volatile("multimem.st.relaxed.sys.global.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(addr), "f"(v.x), "f"(v.y),
                 "f"(v.z), "f"(v.w)
                 : "memory");
}

// Elements [e0, e1) of the flat [K][ld] buffers (multiples of 4), one float4 per thread and
// iteration.  P: this rank's parameters (identical on every rank before the step); M, V: this
// rank's moments for its range (index e - e0); columns >= n are padding: left as they are.
template <bool MC>
__global__ void __launch_bounds__(256) k_reduce_adam_bcast(const float *__restrict__ P, PeerPtrs params, PeerPtrs grads,
                                                           float *p_mc, float *g_mc, float *__restrict__ M,
                                                           float *__restrict__ V, int64_t ld, int64_t n, int64_t e0,
                                                           int64_t e1, int world, AdamArgs a) {
    adam_device_step(a);
    const float4 zero4 = make_float4(0.f, 0.f, 0.f, 0.f);
    for (int64_t e = e0 + 4 * ((int64_t)blockIdx.x * blockDim.x + threadIdx.x); e < e1;
         e += 4 * (int64_t)gridDim.x * blockDim.x) {
        float4 g;
        if (MC) {
            g = mc_ld_reduce(g_mc + e);
        } else {
            g = ld_sys(grads.p[0] + e);
            for (int q = 1; q < world; q++) {
                const float4 o = ld_sys(grads.p[q] + e);
                g.x += o.x;
                g.y += o.y;
                g.z += o.z;
                g.w += o.w;
            }
        }
        const int row = (int)(e / ld);
        const int64_t col = e - (int64_t)row * ld;  // ld % 4 == 0: the float4 stays in one row
        const float lr = a.lr[row_class(row)];
        float4 p = *reinterpret_cast<const float4 *>(P + e);
        const int64_t k = e - e0;
        float4 m = a.sgd ? zero4 : *reinterpret_cast<const float4 *>(M + k);
        float4 v = a.sgd ? zero4 : *reinterpret_cast<const float4 *>(V + k);
        float *pp = &p.x, *gg = &g.x, *mm = &m.x, *vv = &v.x;
#pragma unroll
        for (int c = 0; c < 4; c++)
            if (col + c < n) adam1(pp[c], gg[c], mm[c], vv[c], lr, a);
        if (!a.sgd) {
            *reinterpret_cast<float4 *>(M + k) = m;
            *reinterpret_cast<float4 *>(V + k) = v;
        }
        if (MC) {
            mc_st(p_mc + e, p);
            mc_st(g_mc + e, zero4);
        } else {
            for (int q = 0; q < world; q++) {
                st_sys(params.p[q] + e, p);
                st_sys(grads.p[q] + e, zero4);
            }
        }
    }
}

void comm_shard(int64_t total, int rank, int world, int64_t *e0, int64_t *e1) {
    const int64_t q4 = (total / 4 + world - 1) / world;  // float4s per rank
    *e0 = std::min(total, (int64_t)rank * q4 * 4);
    *e1 = std::min(total, (int64_t)(rank + 1) * q4 * 4);
}

cudaError_t launch_peer_barrier(uint32_t *const *flags, int rank, int world, uint32_t *epoch_dev, int64_t *step_dev,
                                cudaStream_t s) {
    PeerFlags f{};
    for (int q = 0; q < world; q++) f.p[q] = flags[q];
    k_peer_barrier<<<1, 32, 0, s>>>(f, rank, world, epoch_dev, step_dev);
    return cudaGetLastError();
}

cudaError_t launch_reduce_adam_bcast(const gs_params &p, float *const *param_peers, float *const *grad_peers,
                                     float *p_mc, float *g_mc, float *m, float *v, const gs_adam_hparams &hp,
                                     int64_t step, const int64_t *step_dev, int rank, int world, cudaStream_t s) {
    int64_t e0, e1;
    comm_shard((int64_t)gs_param_rows(p.sh_degree) * p.ld, rank, world, &e0, &e1);
    if (e1 <= e0) return cudaGetLastError();
    AdamArgs a = adam_args(hp, step, 1, step_dev);
    PeerPtrs pp{}, gp{};
    for (int q = 0; q < world; q++) {
        pp.p[q] = param_peers[q];
        gp.p[q] = grad_peers[q];
    }
    int sms = 148;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const int64_t need = (e1 - e0 + 4 * 256 - 1) / (4 * 256);
    const unsigned blocks = (unsigned)std::max<int64_t>(1, std::min<int64_t>(need, (int64_t)sms * 8));
    ProfScope prof("k_reduce_adam_bcast", s);
    if (p_mc && g_mc)
        k_reduce_adam_bcast<true><<<blocks, 256, 0, s>>>(p.data, pp, gp, p_mc, g_mc, m, v, p.ld, p.n, e0, e1, world, a);
    else
        k_reduce_adam_bcast<false><<<blocks, 256, 0, s>>>(p.data, pp, gp, nullptr, nullptr, m, v, p.ld, p.n, e0, e1,
                                                          world, a);
    return cudaGetLastError();
}

}  // namespace gsk
