// Multi-GPU z slabs in the library (slab.cuh). The sharded problem keeps the
// reference's solver control flow (optimizer.cpp:113-407 via solvers.cu / cg.cu) and the
// reference's multilevel driver (multilevel.cpp:117-145); only the operators and reductions
// change.
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <cmath>
#include <cstring>
#include <mutex>
#include <stdexcept>
#include <string>

#include "slab.cuh"

namespace mfreg_b200 {

namespace {

__global__ void k_sum3_local(double* d) { d[3] = (d[0] + d[1]) + d[2]; }  // components added in order

__global__ void k_rank_sum(const double* __restrict__ g, int size, int count, double* __restrict__ out) {
    const int k = threadIdx.x;
    if (k >= count) return;
    double v = g[k];
    for (int r = 1; r < size; ++r) v += g[r * count + k];  // rank order: identical on every rank
    out[k] = v;
}

__global__ void k_add(long long n, const double* __restrict__ a, double* __restrict__ o) {
    for (long long i = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
         i += static_cast<long long>(gridDim.x) * blockDim.x)
        o[i] = o[i] + a[i];
}

// ---------------------------------------------------------------- NCCL (loaded at run time)
struct NcclApi {
    decltype(&ncclGetUniqueId) getUniqueId = nullptr;
    decltype(&ncclCommInitRank) commInitRank = nullptr;
    decltype(&ncclCommDestroy) commDestroy = nullptr;
    decltype(&ncclGroupStart) groupStart = nullptr;
    decltype(&ncclGroupEnd) groupEnd = nullptr;
    decltype(&ncclSend) send = nullptr;
    decltype(&ncclRecv) recv = nullptr;
    decltype(&ncclAllGather) allGather = nullptr;
    decltype(&ncclGetErrorString) errorString = nullptr;
};

const NcclApi& nccl() {
    static NcclApi api;
    static std::once_flag once;
    static std::string err;
    std::call_once(once, [] {
        void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
        if (!h) {
            err = std::string("NCCL not available: ") + dlerror();
            return;
        }
        auto sym = [&](auto& f, const char* name) {
            f = reinterpret_cast<std::remove_reference_t<decltype(f)>>(dlsym(h, name));
            if (!f) err = std::string("NCCL symbol missing: ") + name;
        };
        sym(api.getUniqueId, "ncclGetUniqueId");
        sym(api.commInitRank, "ncclCommInitRank");
        sym(api.commDestroy, "ncclCommDestroy");
        sym(api.groupStart, "ncclGroupStart");
        sym(api.groupEnd, "ncclGroupEnd");
        sym(api.send, "ncclSend");
        sym(api.recv, "ncclRecv");
        sym(api.allGather, "ncclAllGather");
        sym(api.errorString, "ncclGetErrorString");
    });
    if (!err.empty()) throw std::runtime_error(err);
    return api;
}

void nccl_check(ncclResult_t r, const char* what) {
    if (r != ncclSuccess) throw std::runtime_error(std::string(what) + ": " + nccl().errorString(r));
}

class NcclComm : public SlabComm {
public:
    NcclComm(const void* id, int nranks, int rank) : rank_(rank), size_(nranks) {
        ncclUniqueId uid;
        std::memcpy(&uid, id, sizeof(uid));
        nccl_check(nccl().commInitRank(&comm_, nranks, uid, rank), "ncclCommInitRank");
    }
    ~NcclComm() override {
        if (comm_) nccl().commDestroy(comm_);
    }
    int rank() const override { return rank_; }
    int size() const override { return size_; }
    bool stream_ordered() const override { return true; }
    void exchange(const std::vector<Msg>& sends, const std::vector<Msg>& recvs, cudaStream_t s) override {
        if (sends.empty() && recvs.empty()) return;
        const auto& N = nccl();
        nccl_check(N.groupStart(), "ncclGroupStart");
        for (const auto& m : sends) nccl_check(N.send(m.buf, m.bytes, ncclChar, m.peer, comm_, s), "ncclSend");
        for (const auto& m : recvs) nccl_check(N.recv(m.buf, m.bytes, ncclChar, m.peer, comm_, s), "ncclRecv");
        nccl_check(N.groupEnd(), "ncclGroupEnd");
    }
    void allgather(const double* in, double* out, int count, cudaStream_t s) override {
        nccl_check(nccl().allGather(in, out, static_cast<std::size_t>(count), ncclDouble, comm_, s), "ncclAllGather");
    }

private:
    ncclComm_t comm_ = nullptr;
    int rank_, size_;
};

}  // namespace

// ---------------------------------------------------------------- in-process ranks
// reusable host barrier (generation counter)
class HostBarrier {
public:
    explicit HostBarrier(int n) : n_(n) {}
    void arrive_and_wait() {
        std::unique_lock<std::mutex> lk(m_);
        const long long gen = gen_;
        if (++count_ == n_) {
            count_ = 0;
            ++gen_;
            cv_.notify_all();
            return;
        }
        cv_.wait(lk, [&] { return gen_ != gen; });
    }

private:
    std::mutex m_;
    std::condition_variable cv_;
    int n_, count_ = 0;
    long long gen_ = 0;
};

class LocalHub {
public:
    explicit LocalHub(int n) : n_(n), bar_(n), box_(static_cast<std::size_t>(n)), gin_(static_cast<std::size_t>(n)) {}
    int n_;
    HostBarrier bar_;
    std::vector<std::vector<SlabComm::Msg>> box_;  // sends posted by each rank
    std::vector<const double*> gin_;               // all-gather inputs
};

namespace {

void peer_copy(void* dst, const void* src, std::size_t bytes, cudaStream_t s) {
    cudaPointerAttributes ad{}, as{};
    MFREG_CUDA(cudaPointerGetAttributes(&ad, dst));
    MFREG_CUDA(cudaPointerGetAttributes(&as, src));
    if (ad.device == as.device) MFREG_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToDevice, s));
    else MFREG_CUDA(cudaMemcpyPeerAsync(dst, ad.device, src, as.device, bytes, s));
}

class LocalComm : public SlabComm {
public:
    LocalComm(std::shared_ptr<LocalHub> hub, int rank) : hub_(std::move(hub)), rank_(rank) {}
    int rank() const override { return rank_; }
    int size() const override { return hub_->n_; }
    bool stream_ordered() const override { return false; }
    void exchange(const std::vector<Msg>& sends, const std::vector<Msg>& recvs, cudaStream_t s) override {
        MFREG_CUDA(cudaStreamSynchronize(s));  // the send buffers are final
        hub_->box_[static_cast<std::size_t>(rank_)] = sends;
        hub_->bar_.arrive_and_wait();
        std::vector<int> taken(static_cast<std::size_t>(hub_->n_), 0);  // k-th receive from p = k-th send of p to me
        for (const auto& m : recvs) {
            const auto& box = hub_->box_[static_cast<std::size_t>(m.peer)];
            int seen = 0;
            const Msg* src = nullptr;
            for (const auto& c : box)
                if (c.peer == rank_ && seen++ == taken[static_cast<std::size_t>(m.peer)]) {
                    src = &c;
                    break;
                }
            if (!src || src->bytes != m.bytes) throw std::logic_error("slab exchange: unmatched message");
            ++taken[static_cast<std::size_t>(m.peer)];
            peer_copy(m.buf, src->buf, m.bytes, s);
        }
        MFREG_CUDA(cudaStreamSynchronize(s));
        hub_->bar_.arrive_and_wait();  // every copy done before a sender reuses its buffer
    }
    void allgather(const double* in, double* out, int count, cudaStream_t s) override {
        MFREG_CUDA(cudaStreamSynchronize(s));
        hub_->gin_[static_cast<std::size_t>(rank_)] = in;
        hub_->bar_.arrive_and_wait();
        for (int r = 0; r < hub_->n_; ++r)
            peer_copy(out + static_cast<std::size_t>(r) * count, hub_->gin_[static_cast<std::size_t>(r)],
                      static_cast<std::size_t>(count) * sizeof(double), s);
        MFREG_CUDA(cudaStreamSynchronize(s));
        hub_->bar_.arrive_and_wait();
    }

private:
    std::shared_ptr<LocalHub> hub_;
    int rank_;
};

}  // namespace

std::unique_ptr<SlabComm> make_nccl_comm(const void* unique_id, int nranks, int rank) {
    if (nranks < 1 || rank < 0 || rank >= nranks) throw std::invalid_argument("nccl comm: bad rank / size");
    return std::make_unique<NcclComm>(unique_id, nranks, rank);
}

void nccl_unique_id(void* out128) {
    ncclUniqueId id;
    nccl_check(nccl().getUniqueId(&id), "ncclGetUniqueId");
    std::memcpy(out128, &id, sizeof(id));
}

std::vector<std::unique_ptr<SlabComm>> make_local_comms(int nranks) {
    if (nranks < 1) throw std::invalid_argument("local comm: nranks must be >= 1");
    auto hub = std::make_shared<LocalHub>(nranks);
    std::vector<std::unique_ptr<SlabComm>> out;
    for (int r = 0; r < nranks; ++r) out.push_back(std::make_unique<LocalComm>(hub, r));
    return out;
}

// ---------------------------------------------------------------- DistSum
DistSum::DistSum(idx_t N, const std::vector<std::vector<Seg>>& segs, int rank) {
    const idx_t C = kChunk;
    nch_ = (N + C - 1) / C;
    const int nr = static_cast<int>(segs.size());
    // per rank: interior chunk partials first (in segment / chunk order), then one C-slot per piece
    struct Piece {
        int r;
        idx_t lo, hi;
        std::size_t slot;
    };
    std::vector<std::vector<std::pair<idx_t, std::size_t>>> interior(nr);  // (chunk, slot)
    std::vector<std::vector<Piece>> pieces(nr);
    std::size_t ni_max = 0, np_max = 0;
    for (int r = 0; r < nr; ++r) {
        for (const Seg& sg : segs[r]) {
            if (sg.b <= sg.a) continue;
            for (idx_t c = sg.a / C; c * C < sg.b; ++c) {
                const idx_t c_lo = c * C, c_hi = std::min(N, c_lo + C);
                const idx_t lo = std::max(sg.a, c_lo), hi = std::min(sg.b, c_hi);
                if (lo == c_lo && hi == c_hi) interior[r].push_back({c, interior[r].size()});
                else pieces[r].push_back({r, lo, hi, 0});
            }
        }
        ni_max = std::max(ni_max, interior[r].size());
        np_max = std::max(np_max, pieces[r].size());
    }
    B_ = std::max<std::size_t>(1, ni_max + np_max * C);
    for (int r = 0; r < nr; ++r)
        for (std::size_t k = 0; k < pieces[r].size(); ++k) pieces[r][k].slot = ni_max + k * C;
    // assembly table: chunk -> interior block entry, or its pieces in index order
    std::vector<long long> off(nch_, -1);
    std::vector<int> cnt(nch_, 0);
    std::vector<std::vector<Piece>> per_chunk(nch_);
    for (int r = 0; r < nr; ++r) {
        for (const auto& [c, slot] : interior[r]) {
            if (off[c] >= 0 || !per_chunk[c].empty()) throw std::invalid_argument("DistSum: overlapping segments");
            off[c] = static_cast<long long>(r) * B_ + slot;
        }
        for (const Piece& pc : pieces[r]) per_chunk[pc.lo / C].push_back(pc);
    }
    std::vector<ChunkPiece> plist;
    for (idx_t c = 0; c < nch_; ++c) {
        auto& v = per_chunk[c];
        if (v.empty()) {
            if (off[c] < 0) throw std::invalid_argument("DistSum: segments do not cover the index space");
            continue;
        }
        if (off[c] >= 0) throw std::invalid_argument("DistSum: overlapping segments");
        std::sort(v.begin(), v.end(), [](const Piece& x, const Piece& y) { return x.lo < y.lo; });
        idx_t at = c * C;
        for (const Piece& pc : v) {
            if (pc.lo != at) throw std::invalid_argument("DistSum: segments do not cover the index space");
            at = pc.hi;
        }
        if (at != std::min(N, (c + 1) * C)) throw std::invalid_argument("DistSum: segments do not cover the index space");
        off[c] = static_cast<long long>(plist.size());
        cnt[c] = static_cast<int>(v.size());
        for (const Piece& pc : v)
            plist.push_back({static_cast<long long>(pc.r) * static_cast<long long>(B_) + static_cast<long long>(pc.slot),
                             static_cast<int>(pc.hi - pc.lo)});
    }
    // my local launches: one partials run per maximal stretch of consecutive interior chunks
    const auto& mine = interior[rank];
    for (std::size_t k = 0; k < mine.size();) {
        std::size_t e = k + 1;
        while (e < mine.size() && mine[e].first == mine[e - 1].first + 1) ++e;
        const idx_t lo = mine[k].first * C, hi = std::min(N, (mine[e - 1].first + 1) * C);
        runs_.push_back({false, lo, hi - lo, mine[k].second});
        k = e;
    }
    for (const Piece& pc : pieces[rank]) runs_.push_back({true, pc.lo, pc.hi - pc.lo, pc.slot});
    off_.resize(std::max<idx_t>(1, nch_));
    cnt_.resize(std::max<idx_t>(1, nch_));
    pieces_.resize(std::max<std::size_t>(1, plist.size()));
    vals_.resize(std::max<idx_t>(1, nch_));
    if (nch_) {
        MFREG_CUDA(cudaMemcpy(off_.get(), off.data(), nch_ * sizeof(long long), cudaMemcpyHostToDevice));
        MFREG_CUDA(cudaMemcpy(cnt_.get(), cnt.data(), nch_ * sizeof(int), cudaMemcpyHostToDevice));
    }
    if (!plist.empty())
        MFREG_CUDA(cudaMemcpy(pieces_.get(), plist.data(), plist.size() * sizeof(ChunkPiece), cudaMemcpyHostToDevice));
}

void DistSum::local(int kind, const double* a, const double* b, double* blk, cudaStream_t s) const {
    for (const Run& r : runs_) {
        const double* ap = a + r.lo;
        const double* bp = b ? b + r.lo : nullptr;
        if (r.terms) launch_sum_terms(kind, r.n, ap, bp, blk + r.slot, s);
        else launch_chunk_partials(kind, r.n, ap, bp, blk + r.slot, s);
    }
}

void DistSum::assemble(const double* gathered, double scale, double* out, cudaStream_t s) {
    launch_chunk_assemble(nch_, off_.get(), cnt_.get(), pieces_.get(), gathered, vals_.get(), scale, out, s);
}

// ---------------------------------------------------------------- SlabProblem
SlabProblem::SlabProblem(const double* R_dev, const double* T_dev, const Grid& image, const Grid& deform, double tau,
                         double rho, double alpha, SlabComm& comm, cudaStream_t s, Mode mode)
    : img_(image), dg_(deform), comm_(comm), s_(s),
      parts_(slab_partition(image, deform, comm.size(), mode == Mode::Parity)), red_(Mode::Fast, 3 * deform.count()),
      sc_(16) {
    if (mode == Mode::Fast32) throw std::invalid_argument("z slabs run in fast or parity mode");
    parity_ = mode == Mode::Parity;
    me_ = parts_[static_cast<std::size_t>(comm.rank())];
    const SlabSpec spec{me_.zlo, me_.zhi, me_.own_lo, me_.own_hi};
    obj_ = std::make_unique<DeviceObjective>(R_dev, T_dev, image, deform, tau, rho, alpha, mode, s, spec);
    if (parity_) {
        const idx_t pl = image.m[0] * image.m[1], pn = deform.m[0] * deform.m[1], ny = deform.count();
        std::vector<std::vector<DistSum::Seg>> sd, ss, sdot;
        for (const SlabInfo& p : parts_) {
            sd.push_back({{p.zlo * pl, p.zhi * pl}});
            ss.push_back({{p.own_lo * pn, p.own_hi * pn}});
            sdot.push_back({});
            for (int d = 0; d < 3; ++d) sdot.back().push_back({d * ny + p.own_lo * pn, d * ny + p.own_hi * pn});
        }
        dsD_ = DistSum(image.count(), sd, comm.rank());
        dsS_ = DistSum(ny, ss, comm.rank());
        dsDot_ = DistSum(3 * ny, sdot, comm.rank());
        const std::size_t B = std::max({dsD_.block(), dsS_.block(), dsDot_.block()});
        blk_.resize(B);
        gat_.resize(B * static_cast<std::size_t>(comm.size()));
    }
    sc_dev_.resize(16);
    gath_.resize(static_cast<std::size_t>(4 * comm.size()));
    const int bnd_in = comm.rank() > 0 ? parts_[static_cast<std::size_t>(comm.rank() - 1)].bnd : 0;
    stage_.resize(static_cast<std::size_t>(std::max(1, bnd_in) * dg_.m[0] * dg_.m[1] * 3));
}

SlabProblem::~SlabProblem() = default;

void SlabProblem::halo(const double* v) {
    const int r = comm_.rank(), n = comm_.size();
    const idx_t pn = dg_.m[0] * dg_.m[1];
    std::vector<SlabComm::Msg> sends, recvs;
    auto add = [&](std::vector<SlabComm::Msg>& list, int peer, int lo, int hi) {
        if (hi <= lo) return;
        for (int d = 0; d < 3; ++d)
            list.push_back({peer, planes(v, d, lo), static_cast<std::size_t>((hi - lo) * pn) * sizeof(double)});
    };
    if (r > 0) {
        const SlabInfo& lo = parts_[static_cast<std::size_t>(r - 1)];
        add(sends, r - 1, me_.own_lo, lo.need_hi);
        add(recvs, r - 1, me_.need_lo, me_.own_lo);
    }
    if (r + 1 < n) {
        const SlabInfo& up = parts_[static_cast<std::size_t>(r + 1)];
        add(sends, r + 1, up.need_lo, me_.own_hi);
        add(recvs, r + 1, me_.own_hi, me_.need_hi);
    }
    comm_.exchange(sends, recvs, s_);
}

void SlabProblem::boundary(double* q) {
    const int r = comm_.rank(), n = comm_.size();
    const idx_t pn = dg_.m[0] * dg_.m[1];
    std::vector<SlabComm::Msg> sends, recvs;
    if (r + 1 < n && me_.bnd)
        for (int d = 0; d < 3; ++d)
            sends.push_back({r + 1, planes(q, d, me_.own_hi), static_cast<std::size_t>(me_.bnd * pn) * sizeof(double)});
    const int bin = r > 0 ? parts_[static_cast<std::size_t>(r - 1)].bnd : 0;
    if (bin)
        for (int d = 0; d < 3; ++d)
            recvs.push_back({r - 1, stage_.get() + d * bin * pn, static_cast<std::size_t>(bin * pn) * sizeof(double)});
    comm_.exchange(sends, recvs, s_);
    if (bin)
        for (int d = 0; d < 3; ++d) {
            note_launch();
            k_add<<<static_cast<unsigned>(std::min<idx_t>((bin * pn + 255) / 256, 1184)), 256, 0, s_>>>(
                bin * pn, stage_.get() + d * bin * pn, planes(q, d, me_.own_lo));
        }
    check_launch("slab boundary");
}

void SlabProblem::rank_sum(const double* gathered, int count, double* out) {
    note_launch();
    k_rank_sum<<<1, 32, 0, s_>>>(gathered, comm_.size(), count, out);
}

void SlabProblem::dist_sum(DistSum& ds, int kind, const double* a, const double* b, double scale, double* out_dev) {
    ds.local(kind, a, b, blk_.get(), s_);
    comm_.allgather(blk_.get(), gat_.get(), static_cast<int>(ds.block()), s_);
    ds.assemble(gat_.get(), scale, out_dev, s_);
    check_launch("slab chunked sum");
}

double SlabProblem::eval(const double* y, double* grad) {
    if (parity_) {  // optimizer.cpp:64-92 with the reference's reductions across ranks
        halo(y);
        obj_->parity_eval_local(y, grad);
        const idx_t ny = dg_.count();
        dist_sum(dsD_, SUM_ONE_MINUS_SQ, obj_->parity_r(), nullptr, img_.cell_volume(), sc_.dev(0));  // ngf.cpp:225-231
        for (int d = 0; d < 3; ++d)  // curvature.cpp:31-45, per component
            dist_sum(dsS_, SUM_SQ, obj_->lap_u() + d * ny, nullptr, 1.0, sc_dev_.get() + 12 + d);
        launch_curv_finalize(sc_dev_.get() + 12, dg_.cell_volume(), obj_->alpha(), sc_.dev(1), s_);
        check_launch("slab eval (parity)");
        const double* v = sc_.fetch(2, s_);
        last_d_ = v[0];
        last_s_ = v[1];
        return last_d_ + last_s_;
    }
    halo(y);
    obj_->eval(y, grad);
    if (grad) boundary(grad);  // (fast mode)
    const double loc[2] = {obj_->last_distance(), obj_->last_regularizer()};
    MFREG_CUDA(cudaMemcpyAsync(sc_dev_.get() + 8, loc, sizeof(loc), cudaMemcpyHostToDevice, s_));
    comm_.allgather(sc_dev_.get() + 8, gath_.get(), 2, s_);
    rank_sum(gath_.get(), 2, sc_.dev(0));
    const double* v = sc_.fetch(2, s_);
    last_d_ = v[0];
    last_s_ = v[1];
    return last_d_ + last_s_;
}

void SlabProblem::gn_hessian_vec(const double* p, double* q) {
    halo(p);
    obj_->gn_hessian_vec(p, q);
    if (!parity_) boundary(q);  // (parity: each owned node's gather ran complete here)
}

void SlabProblem::seed_hessian_vec(const double* p, double gamma, double* q) {
    halo(p);  // the +-2-plane curvature stencil of the owned planes
    obj_->seed_hessian_vec(p, gamma, q);
}

void SlabProblem::local_dot(const double* a, const double* b, double* dev) {
    const idx_t ny = dg_.count(), pn = dg_.m[0] * dg_.m[1], off = me_.own_lo * pn;
    const idx_t cnt = (me_.own_hi - me_.own_lo) * pn;
    for (int d = 0; d < 3; ++d) red_.sum(SUM_DOT, cnt, a + d * ny + off, b + d * ny + off, dev + d, 1.0, s_);
    note_launch();
    k_sum3_local<<<1, 1, 0, s_>>>(dev);
}

void SlabProblem::dot_async(const double* a, const double* b, double* out_dev) {
    if (parity_) {  // optimizer.cpp:12-19: one chunked sum over the 3 m^y elements
        dist_sum(dsDot_, SUM_DOT, a, b, 1.0, out_dev);
        return;
    }
    local_dot(a, b, sc_dev_.get());
    comm_.allgather(sc_dev_.get() + 3, gath_.get(), 1, s_);
    rank_sum(gath_.get(), 1, out_dev);
    check_launch("slab dot");
}

double SlabProblem::dot(const double* a, const double* b) {
    dot_async(a, b, sc_.dev(2));
    return sc_.fetch(3, s_)[2];
}

double SlabProblem::inf_norm(const double* a, double scale) {
    const idx_t ny = dg_.count(), pn = dg_.m[0] * dg_.m[1], off = me_.own_lo * pn;
    const idx_t cnt = (me_.own_hi - me_.own_lo) * pn;
    for (int d = 0; d < 3; ++d) launch_inf_norm(cnt, a + d * ny + off, scale, sc_dev_.get() + 4 + d, s_);
    check_launch("slab inf_norm");
    comm_.allgather(sc_dev_.get() + 4, gath_.get(), 3, s_);
    std::vector<double> h(static_cast<std::size_t>(3 * comm_.size()));
    MFREG_CUDA(cudaMemcpyAsync(h.data(), gath_.get(), h.size() * sizeof(double), cudaMemcpyDeviceToHost, s_));
    MFREG_CUDA(cudaStreamSynchronize(s_));
    return *std::max_element(h.begin(), h.end());
}

void SlabProblem::gather_full(double* v) {
    const int r = comm_.rank(), n = comm_.size();
    const idx_t pn = dg_.m[0] * dg_.m[1];
    std::vector<SlabComm::Msg> sends, recvs;
    for (int p = 0; p < n; ++p) {
        if (p == r) continue;
        const SlabInfo& o = parts_[static_cast<std::size_t>(p)];
        for (int d = 0; d < 3; ++d) {
            sends.push_back({p, planes(v, d, me_.own_lo), static_cast<std::size_t>((me_.own_hi - me_.own_lo) * pn) * sizeof(double)});
            recvs.push_back({p, planes(v, d, o.own_lo), static_cast<std::size_t>((o.own_hi - o.own_lo) * pn) * sizeof(double)});
        }
    }
    comm_.exchange(sends, recvs, s_);
}

// ---------------------------------------------------------------- sharded multilevel driver
MultilevelResult register_multilevel_slabs(const double* R_dev, const double* T_dev, const Grid& image,
                                           const MultilevelConfig& cfg, SlabComm& comm, cudaStream_t s) {
    if (cfg.mode == Mode::Fast32) throw std::invalid_argument("z slabs run in fast or parity mode");
    if (cfg.levels < 1) throw std::invalid_argument("build_pyramid: levels must be >= 1");
    validate_grid(image, false);
    for (int a = 0; a < 3; ++a) {  // multilevel.cpp:13-29
        idx_t m = image.m[a];
        for (int l = 1; l < cfg.levels; ++l) {
            if (m < 2) throw std::invalid_argument("build_pyramid: too many levels for this size");
            m = (m + 1) / 2;
        }
        if (m < 2) throw std::invalid_argument("build_pyramid: too many levels for this size");
    }
    std::vector<Grid> G(static_cast<std::size_t>(cfg.levels));
    std::vector<DVec> R(static_cast<std::size_t>(cfg.levels)), T(static_cast<std::size_t>(cfg.levels));
    G[0] = image;
    for (int l = 1; l < cfg.levels; ++l) {  // the (replicated) pyramid: every rank downsamples R, T
        for (int a = 0; a < 3; ++a) {
            G[l].m[a] = (G[l - 1].m[a] + 1) / 2;
            G[l].h[a] = 2.0 * G[l - 1].h[a];
        }
        R[l].resize(static_cast<std::size_t>(G[l].count()));
        T[l].resize(static_cast<std::size_t>(G[l].count()));
        launch_downsample(G[l - 1], G[l], l == 1 ? R_dev : R[l - 1].get(), R[l].get(), s);
        launch_downsample(G[l - 1], G[l], l == 1 ? T_dev : T[l - 1].get(), T[l].get(), s);
    }
    check_launch("build_pyramid");
    MultilevelResult out;
    DVec y;
    Grid prev{};
    bool have_prev = false;
    for (int l = cfg.levels - 1; l >= 0; --l) {
        const Grid dg = deformation_grid_for(G[l], cfg.deform_ratio);
        const double* rp = l == 0 ? R_dev : R[l].get();
        const double* tp = l == 0 ? T_dev : T[l].get();
        const idx_t n = 3 * dg.count();
        DVec y0(static_cast<std::size_t>(n)), yl(static_cast<std::size_t>(n));
        bool sharded = comm.size() > 1;
        if (sharded) {
            try {
                (void)slab_partition(G[l], dg, comm.size(), cfg.mode == Mode::Parity);
            } catch (const std::invalid_argument&) {
                sharded = false;  // too thin for the slab halo: this level runs replicated
            }
        }
        MinimizeResult res;
        if (sharded) {
            SlabProblem P(rp, tp, G[l], dg, cfg.tau, cfg.rho, cfg.alpha, comm, s, cfg.mode);
            if (have_prev) launch_prolong(prev, dg, y.get(), y0.get(), s);
            else MFREG_CUDA(cudaMemcpyAsync(y0.get(), P.identity_dev(), n * sizeof(double), cudaMemcpyDeviceToDevice, s));
            res = cfg.method == Method::Lbfgs ? lbfgs_minimize(P, y0.get(), yl.get(), cfg.opt)
                                              : gauss_newton_minimize(P, y0.get(), yl.get(), cfg.opt);
            P.gather_full(yl.get());  // every rank holds the level's whole result (prolongation input)
        } else {
            DeviceObjective obj(rp, tp, G[l], dg, cfg.tau, cfg.rho, cfg.alpha, cfg.mode, s);
            if (have_prev) launch_prolong(prev, dg, y.get(), y0.get(), s);
            else MFREG_CUDA(cudaMemcpyAsync(y0.get(), obj.identity_dev(), n * sizeof(double), cudaMemcpyDeviceToDevice, s));
            res = cfg.method == Method::Lbfgs ? lbfgs_minimize(obj, y0.get(), yl.get(), cfg.opt)
                                              : gauss_newton_minimize(obj, y0.get(), yl.get(), cfg.opt);
        }
        check_launch("prolong");
        MFREG_CUDA(cudaStreamSynchronize(s));
        LevelResult lr{G[l], dg, std::move(res), DVec()};
        if (cfg.keep_level_y) {
            lr.y.resize(static_cast<std::size_t>(n));
            MFREG_CUDA(cudaMemcpyAsync(lr.y.get(), yl.get(), n * sizeof(double), cudaMemcpyDeviceToDevice, s));
        }
        y = std::move(yl);
        out.levels.push_back(std::move(lr));
        prev = dg;
        have_prev = true;
    }
    out.y = std::move(y);
    out.deform_grid = prev;
    return out;
}

}  // namespace mfreg_b200

// ---------------------------------------------------------------- C ABI (include/mfreg_cuda.h, "z slabs")
#include "capi_util.cuh"

struct mfreg_cu_comm {
    std::unique_ptr<mfreg_b200::SlabComm> c;
};
struct mfreg_cu_slab {
    mfreg_b200::Grid img, dg;
    mfreg_b200::DVec R, T;
    std::unique_ptr<mfreg_b200::SlabProblem> p;
};

using namespace mfreg_b200;
using namespace mfreg_b200::capi;

extern "C" {

int mfreg_cu_comm_nccl_unique_id(unsigned char out[128]) {
    return guard([&] { nccl_unique_id(out); });
}
int mfreg_cu_comm_create_nccl(const unsigned char id[128], int nranks, int rank, mfreg_cu_comm** out) {
    return guard([&] {
        auto h = std::make_unique<mfreg_cu_comm>();
        h->c = make_nccl_comm(id, nranks, rank);
        *out = h.release();
    });
}
int mfreg_cu_comm_create_local(int nranks, mfreg_cu_comm** out) {
    return guard([&] {
        auto comms = make_local_comms(nranks);
        for (int r = 0; r < nranks; ++r) {
            out[r] = new mfreg_cu_comm;
            out[r]->c = std::move(comms[static_cast<std::size_t>(r)]);
        }
    });
}
int mfreg_cu_comm_destroy(mfreg_cu_comm* c) {
    return guard([&] { delete c; });
}
int mfreg_cu_comm_rank(mfreg_cu_comm* c, int* rank, int* size) {
    return guard([&] {
        *rank = c->c->rank();
        *size = c->c->size();
    });
}

int mfreg_cu_slab_create(mfreg_cu_comm* comm, const double* ref, const double* tpl, const mfreg_cu_grid* image,
                         const mfreg_cu_grid* deform, double tau, double rho, double alpha, int mode, int where,
                         mfreg_cu_slab** out) {
    return guard([&] {
        if (!comm) throw std::invalid_argument("null communicator");
        check_where(where);
        auto h = std::make_unique<mfreg_cu_slab>();
        h->img = to_grid(image);
        h->dg = to_grid(deform);
        validate_grid(h->img, false);
        const std::size_t n = static_cast<std::size_t>(h->img.count());
        h->R.resize(n);
        h->T.resize(n);
        const auto kind = where == MFREG_CU_HOST ? cudaMemcpyHostToDevice : cudaMemcpyDeviceToDevice;
        MFREG_CUDA(cudaMemcpyAsync(h->R.get(), ref, n * sizeof(double), kind, kStream));
        MFREG_CUDA(cudaMemcpyAsync(h->T.get(), tpl, n * sizeof(double), kind, kStream));
        h->p = std::make_unique<SlabProblem>(h->R.get(), h->T.get(), h->img, h->dg, tau, rho, alpha, *comm->c, kStream,
                                             to_mode(mode));
        MFREG_CUDA(cudaStreamSynchronize(kStream));
        *out = h.release();
    });
}
int mfreg_cu_slab_destroy(mfreg_cu_slab* s) {
    return guard([&] { delete s; });
}
int mfreg_cu_slab_info(mfreg_cu_slab* s, int32_t info[7]) {
    return guard([&] {
        const SlabInfo& i = s->p->info();
        const int32_t v[7] = {i.zlo, i.zhi, i.own_lo, i.own_hi, i.need_lo, i.need_hi, i.bnd};
        std::memcpy(info, v, sizeof(v));
    });
}
int mfreg_cu_slab_identity(mfreg_cu_slab* s, double* out) {
    return guard([&] {
        MFREG_CUDA(cudaMemcpyAsync(out, s->p->identity_dev(), s->p->dof() * sizeof(double), cudaMemcpyDeviceToDevice,
                                   kStream));
        MFREG_CUDA(cudaStreamSynchronize(kStream));
    });
}
int mfreg_cu_slab_eval(mfreg_cu_slab* s, double* y, double* grad, double* j) {
    return guard([&] { *j = s->p->eval(y, grad); });
}
int mfreg_cu_slab_last(mfreg_cu_slab* s, double* distance, double* regularizer) {
    return guard([&] {
        *distance = s->p->last_distance();
        *regularizer = s->p->last_regularizer();
    });
}
int mfreg_cu_slab_gn_hessian_vec(mfreg_cu_slab* s, double* p, double* q) {
    return guard([&] {
        s->p->gn_hessian_vec(p, q);
        MFREG_CUDA(cudaStreamSynchronize(kStream));
    });
}
int mfreg_cu_slab_dot(mfreg_cu_slab* s, const double* a, const double* b, double* out) {
    return guard([&] { *out = s->p->dot(a, b); });
}
int mfreg_cu_slab_gather(mfreg_cu_slab* s, double* v) {
    return guard([&] {
        s->p->gather_full(v);
        MFREG_CUDA(cudaStreamSynchronize(kStream));
    });
}
int mfreg_cu_slab_minimize(mfreg_cu_slab* s, int method, const double* y0, const mfreg_cu_opt_config* cfg,
                           double* y_out, mfreg_cu_iter_record* trace, int cap, int* ntrace, int* line_search_failed) {
    return guard([&] {
        if (method != MFREG_CU_LBFGS && method != MFREG_CU_GAUSS_NEWTON) throw std::invalid_argument("unknown method");
        const OptimizerConfig c = to_cfg(cfg);
        const MinimizeResult res = method == MFREG_CU_LBFGS ? lbfgs_minimize(*s->p, y0, y_out, c)
                                                            : gauss_newton_minimize(*s->p, y0, y_out, c);
        s->p->gather_full(y_out);
        MFREG_CUDA(cudaStreamSynchronize(kStream));
        const int n = copy_trace(res.trace, trace, cap);
        if (ntrace) *ntrace = n;
        if (line_search_failed) *line_search_failed = res.line_search_failed ? 1 : 0;
    });
}
int mfreg_cu_slab_register_multilevel(mfreg_cu_comm* comm, const double* ref, const double* tpl,
                                      const mfreg_cu_grid* image, const mfreg_cu_ml_config* cfg, double* y_out,
                                      mfreg_cu_grid* deform_out, mfreg_cu_iter_record* trace, int cap, int* level_iters,
                                      int* line_search_failed, int where) {
    return guard([&] {
        if (!comm) throw std::invalid_argument("null communicator");
        const Grid g = to_grid(image);
        validate_grid(g, false);
        const idx_t n = g.count();
        In r(ref, n, where, kStream), t(tpl, n, where, kStream);
        MultilevelConfig mc;
        mc.levels = cfg->levels;
        mc.deform_ratio = cfg->deform_ratio;
        mc.tau = cfg->tau;
        mc.rho = cfg->rho;
        mc.alpha = cfg->alpha;
        mc.method = cfg->method == MFREG_CU_GAUSS_NEWTON ? Method::GaussNewton : Method::Lbfgs;
        mc.mode = to_mode(cfg->mode);
        mc.opt = to_cfg(&cfg->opt);
        MultilevelResult res = register_multilevel_slabs(r.ptr, t.ptr, g, mc, *comm->c, kStream);
        if (deform_out) from_grid(res.deform_grid, deform_out);
        if (y_out)
            MFREG_CUDA(cudaMemcpyAsync(y_out, res.y.get(), res.y.size() * sizeof(double),
                                       where == MFREG_CU_HOST ? cudaMemcpyDeviceToHost : cudaMemcpyDeviceToDevice,
                                       kStream));
        MFREG_CUDA(cudaStreamSynchronize(kStream));
        int off = 0;
        for (std::size_t l = 0; l < res.levels.size(); ++l) {
            const int k = copy_trace(res.levels[l].result.trace, trace ? trace + std::min(off, cap) : nullptr,
                                     std::max(0, cap - off));
            if (level_iters) level_iters[l] = k;
            if (line_search_failed) line_search_failed[l] = res.levels[l].result.line_search_failed ? 1 : 0;
            off += k;
        }
    });
}

}  // extern "C"
