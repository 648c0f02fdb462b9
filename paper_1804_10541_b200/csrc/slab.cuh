// Multi-GPU z-slab decomposition in the library: communicators, the sharded
// problem the device-resident solvers drive, and the sharded multilevel driver.
//
// One rank per GPU. Rank r evaluates the image planes [zlo, zhi) of slab_partition and owns
// the nodal planes [own_lo, own_hi); solver vectors are full-length nodal vectors of which
// the owned planes are authoritative. Per operator application the only traffic is
//   * the operand's halo planes [need_lo, own_lo) / [own_hi, need_hi) from ranks r-1 / r+1,
//   * the P^T planes [own_hi, own_hi + bnd) a rank shares with r+1 (added on the owner, own
//     + neighbour, a fixed order), and
//   * one all-gather of 1-3 scalars (D, alpha S, a dot product), summed in rank order, so
//     every rank holds bit-identical scalars and takes identical solver branches.
// R and T are replicated (the warp samples T anywhere), so there is no image-grid exchange.
#pragma once

#include <condition_variable>
#include <memory>
#include <mutex>
#include <vector>

#include "kernels.cuh"
#include "objective.cuh"

namespace mfreg_b200 {

// Point-to-point plane exchange + scalar all-gather between the ranks of one job.
class SlabComm {
public:
    struct Msg {
        int peer;
        void* buf;  // device memory
        std::size_t bytes;
    };
    virtual ~SlabComm() = default;
    virtual int rank() const = 0;
    virtual int size() const = 0;
    // every send and receive of one step, ordered on stream s (complete on s afterwards)
    virtual void exchange(const std::vector<Msg>& sends, const std::vector<Msg>& recvs, cudaStream_t s) = 0;
    // out[r * count + k] = rank r's in[k] (device buffers), ordered on s
    virtual void allgather(const double* in, double* out, int count, cudaStream_t s) = 0;
    // true when exchange/allgather are pure stream work (no host synchronisation)
    virtual bool stream_ordered() const = 0;
};

// NCCL over NVLink / NVSwitch (libnccl.so.2 is loaded at run time): ncclSend / ncclRecv in one
// group per step, ncclAllGather for the scalars.
std::unique_ptr<SlabComm> make_nccl_comm(const void* unique_id, int nranks, int rank);
void nccl_unique_id(void* out128);

// N ranks as threads of one process (one or several devices): copies between the ranks'
// device buffers with host barriers. Tests and single-GPU runs of the sharded path.
class LocalHub;
std::vector<std::unique_ptr<SlabComm>> make_local_comms(int nranks);

// chunked_sum (parallel.cpp:51-73) over a global index space [0, N) whose indices are split
// between ranks (each rank: ascending disjoint segments; together they cover [0, N) once), with
// the reference's exact result: every chunk is the sequential sum of its 4096 terms from 0.0 and
// the chunks are added in order. A rank contributes the partials of the chunks inside one of its
// segments and the raw terms of the chunks it owns only part of; after an all-gather of the
// fixed-size blocks every rank assembles the same bits.
class DistSum {
public:
    struct Seg {
        idx_t a, b;
    };
    DistSum() = default;
    DistSum(idx_t N, const std::vector<std::vector<Seg>>& segs, int rank);
    std::size_t block() const { return B_; }  // doubles per rank block
    // my block: interior chunk partials and piece terms of sum_term(kind, a, b, i), a / b
    // indexed globally
    void local(int kind, const double* a, const double* b, double* blk, cudaStream_t s) const;
    // out = scale * sum over chunks in order, from the rank-major gathered blocks
    void assemble(const double* gathered, double scale, double* out, cudaStream_t s);

private:
    struct Run {  // a launch of my local part
        bool terms;
        idx_t lo, n;       // global index range
        std::size_t slot;  // offset in my block
    };
    idx_t nch_ = 0;
    std::size_t B_ = 0;
    std::vector<Run> runs_;
    DevArray<long long> off_;
    DevArray<int> cnt_;
    DevArray<ChunkPiece> pieces_;
    DVec vals_;
};

// One rank's share of the objective as a DeviceProblem: the device-resident
// gauss_newton_minimize / lbfgs_minimize / cg_solve run sharded on it unchanged.
//   fast mode: the fused kernels on the rank's window; shared P^T planes summed on the owner;
//     scalars (D, alpha S, dots) summed in rank order (bit-identical on every rank, within the
//     fast-mode tolerance of the single-GPU objective);
//   parity mode: every quantity bitwise the single-GPU parity objective's (= the reference's):
//     the rank recomputes the per-voxel terms of the nodal slab below its first owned plane
//     from the operand halo, so each owned node's P^T gather runs complete in the reference's
//     red-black order on one rank, and D, S and every vec_dot are the reference's 4096-chunk
//     sums across ranks (DistSum).
class SlabProblem : public DeviceProblem {
public:
    SlabProblem(const double* R_dev, const double* T_dev, const Grid& image, const Grid& deform, double tau,
                double rho, double alpha, SlabComm& comm, cudaStream_t s, Mode mode = Mode::Fast);
    ~SlabProblem() override;
    idx_t dof() const override { return 3 * dg_.count(); }
    // y / p are full-length nodal vectors valid on the owned planes; their halo planes are
    // overwritten with the neighbours' values (scratch planes of a solver vector)
    double eval(const double* y, double* grad) override;
    void gn_hessian_vec(const double* p, double* q) override;
    void seed_hessian_vec(const double* p, double gamma, double* q) override;
    double min_spacing() const override { return obj_->min_spacing(); }
    double alpha() const override { return obj_->alpha(); }
    double last_distance() const override { return last_d_; }
    double last_regularizer() const override { return last_s_; }
    double dot(const double* a, const double* b) override;
    double inf_norm(const double* a, double scale) override;
    cudaStream_t stream() const override { return s_; }
    void dot_async(const double* a, const double* b, double* out_dev) override;
    bool fast_reductions() const override { return false; }
    const SlabInfo& info() const { return me_; }
    const std::vector<SlabInfo>& parts() const { return parts_; }
    const Grid& deform_grid() const { return dg_; }
    const double* identity_dev() const { return obj_->identity_dev(); }
    // every rank's owned planes of v into v (full vector valid on every rank)
    void gather_full(double* v);

private:
    void halo(const double* v);
    void boundary(double* q);
    double* planes(const double* v, int d, int lo) const {
        return const_cast<double*>(v) + d * dg_.count() + static_cast<idx_t>(lo) * dg_.m[0] * dg_.m[1];
    }
    // local owned-plane partial of <a, b> (components added in order) into dev[0]
    void local_dot(const double* a, const double* b, double* dev);
    void rank_sum(const double* gathered, int count, double* out);  // out[k] = sum_r g[r*count+k], rank order
    Grid img_, dg_;
    SlabComm& comm_;
    cudaStream_t s_;
    std::vector<SlabInfo> parts_;
    SlabInfo me_{};
    std::unique_ptr<DeviceObjective> obj_;
    bool parity_ = false;
    DistSum dsD_, dsS_, dsDot_;  // parity: D over the image, S per component, vec_dot over 3 m^y
    DVec blk_, gat_;
    // parity: my block of ds, all-gathered, assembled into out_dev (scale * chunked_sum)
    void dist_sum(DistSum& ds, int kind, const double* a, const double* b, double scale, double* out_dev);
    Reducer red_;
    DVec stage_, sc_dev_, gath_;
    Scalars sc_;
    double last_d_ = 0.0, last_s_ = 0.0;
};

// register_multilevel (multilevel.cpp:117-145) over z slabs: every level sharded across the
// communicator's ranks (a level too thin for the slab halo runs replicated on every rank);
// the coarse result is gathered to every rank before the prolongation. Fast mode.
MultilevelResult register_multilevel_slabs(const double* R_dev, const double* T_dev, const Grid& image,
                                           const MultilevelConfig& cfg, SlabComm& comm, cudaStream_t s);

}  // namespace mfreg_b200
