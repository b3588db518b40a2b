// pcop-b200 — header-only C++17 wrapper over the C ABI (pcb.h) with the shape of the
// reference's pcop::ProductConvolutionOperator (pc_operator.hpp:17-66).
//
//   PCB_EINVAL      -> std::invalid_argument (reference messages, pc_operator.cpp:34-37,46,59-60,86)
//   other failures  -> std::runtime_error
// Vectors are std::vector<double> in the domain's lexicographic order (last axis fastest).
#ifndef PCB_OPERATOR_HPP
#define PCB_OPERATOR_HPP

#include <cstdint>
#include <new>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "pcb/pcb.h"

namespace pcb {

using Point = std::vector<int64_t>;

struct Box {
    Point lo, hi;  // inclusive (box.hpp:22-30)
    int64_t num_points() const {
        int64_t n = 1;
        for (size_t i = 0; i < lo.size(); ++i) n *= hi[i] - lo[i] + 1;
        return n;
    }
};

// A dense field on a box, zero outside (grid_function.hpp:14-67).
struct Field {
    Box box;
    std::vector<double> values;
};

inline void check(pcb_status st) {
    if (st == PCB_OK) return;
    const std::string msg = pcb_last_error();
    if (st == PCB_EINVAL) throw std::invalid_argument(msg);
    throw std::runtime_error(msg);
}

// std::allocator over page-locked host memory (pcb_host_alloc): vectors allocated with it go
// straight to the copy engines in apply_batch (no bounce staging).
template <typename T>
struct pinned_allocator {
    using value_type = T;
    pinned_allocator() = default;
    template <typename U>
    pinned_allocator(const pinned_allocator<U>&) {}
    T* allocate(size_t n) {
        void* p = nullptr;
        if (pcb_host_alloc(static_cast<uint64_t>(n) * sizeof(T), &p) != PCB_OK) throw std::bad_alloc();
        return static_cast<T*>(p);
    }
    void deallocate(T* p, size_t) { pcb_host_free(p); }
    template <typename U>
    bool operator==(const pinned_allocator<U>&) const { return true; }
    template <typename U>
    bool operator!=(const pinned_allocator<U>&) const { return false; }
};
using pinned_vector = std::vector<double, pinned_allocator<double>>;

// Page-locks a buffer the caller owns for the guard's lifetime (pcb_host_register): an ordinary
// std::vector<double> that is applied many times then goes straight to the copy engines.
class host_registration {
  public:
    host_registration(const double* p, size_t n) : p_(const_cast<double*>(p)) {
        if (n == 0) p_ = nullptr;
        else check(pcb_host_register(p_, static_cast<uint64_t>(n) * sizeof(double)));
    }
    explicit host_registration(const std::vector<double>& v) : host_registration(v.data(), v.size()) {}
    ~host_registration() {
        if (p_) pcb_host_unregister(p_);
    }
    host_registration(const host_registration&) = delete;
    host_registration& operator=(const host_registration&) = delete;

  private:
    double* p_;
};

// A fresh 128-byte NCCL id for pcb_options.nccl_id (shard-by-k with the reduce inside the
// library): create it on one rank and send it to the others (MPI_Bcast, a file, a socket ...).
inline std::vector<unsigned char> comm_unique_id() {
    std::vector<unsigned char> id(128);
    check(pcb_comm_unique_id(id.data()));
    return id;
}

// Options of one shard of a k-sharded operator: this process owns the cost-balanced
// block `rank` of `count`; with `nccl_id` every apply sums the shards' partials over NCCL
// (`reduce`: PCB_REDUCE_ALL -> every rank gets the full result, PCB_REDUCE_ROOT -> rank 0).
inline pcb_options shard_options(int32_t rank, int32_t count, const std::vector<unsigned char>* nccl_id = nullptr,
                                 int32_t reduce = PCB_REDUCE_ALL, int32_t device = -1) {
    pcb_options o;
    pcb_default_options(&o);
    o.shard_rank = rank;
    o.shard_count = count;
    o.device = device;
    if (nccl_id) {
        o.nccl_id = nccl_id->data();
        o.reduce = reduce;
    }
    return o;
}

class ProductConvolutionOperator {
  public:
    ProductConvolutionOperator(const Box& domain, const std::vector<Field>& weights,
                               const std::vector<Field>& impulses, const pcb_options* opt = nullptr)
        : domain_(domain) {
        if (weights.size() != impulses.size())
            throw std::invalid_argument("PCOp: one weight per impulse required");
        const int32_t d = static_cast<int32_t>(domain.lo.size());
        std::vector<int64_t> wl, wh, pl, ph;
        std::vector<const double*> wv, pv;
        for (size_t k = 0; k < weights.size(); ++k) {
            wl.insert(wl.end(), weights[k].box.lo.begin(), weights[k].box.lo.end());
            wh.insert(wh.end(), weights[k].box.hi.begin(), weights[k].box.hi.end());
            pl.insert(pl.end(), impulses[k].box.lo.begin(), impulses[k].box.lo.end());
            ph.insert(ph.end(), impulses[k].box.hi.begin(), impulses[k].box.hi.end());
            wv.push_back(weights[k].values.data());
            pv.push_back(impulses[k].values.data());
        }
        check(pcb_create(d, domain.lo.data(), domain.hi.data(), static_cast<int32_t>(weights.size()), nullptr,
                         wl.data(), wh.data(), wv.data(), pl.data(), ph.data(), pv.data(), opt, &op_));
    }
    ~ProductConvolutionOperator() { pcb_destroy(op_); }
    ProductConvolutionOperator(const ProductConvolutionOperator&) = delete;
    ProductConvolutionOperator& operator=(const ProductConvolutionOperator&) = delete;
    ProductConvolutionOperator(ProductConvolutionOperator&& o) noexcept : domain_(std::move(o.domain_)), op_(o.op_) {
        o.op_ = nullptr;
    }

    const Box& domain() const { return domain_; }
    pcb_info info() const {
        pcb_info i{};
        check(pcb_get_info(op_, &i));
        return i;
    }

    // pc_operator.cpp:45-56
    std::vector<double> apply(const std::vector<double>& f) const { return run(f, 1, false); }
    // pc_operator.cpp:58-69
    std::vector<double> apply_adjoint(const std::vector<double>& f) const { return run(f, 1, true); }
    // B vectors, vector-major
    std::vector<double> apply_batch(const std::vector<double>& F, int32_t B) const { return run(F, B, false); }
    // pinned buffers (pinned_vector): no bounce staging on either side
    void apply_batch(const pinned_vector& F, pinned_vector& G, int32_t B, bool adjoint = false) const {
        const int64_t N = domain_.num_points();
        if (static_cast<int64_t>(F.size()) != N * B)
            throw std::invalid_argument(adjoint ? "PCOp::apply_adjoint: shape mismatch" : "PCOp::apply: shape mismatch");
        G.resize(F.size());
        check(adjoint ? pcb_apply_adjoint_batch(op_, B, F.data(), G.data()) : pcb_apply_batch(op_, B, F.data(), G.data()));
    }
    // caller-owned output (G is not resized: buffers page-locked with host_registration stay put)
    void apply_batch(const std::vector<double>& F, std::vector<double>& G, int32_t B, bool adjoint = false) const {
        const int64_t N = domain_.num_points();
        if (static_cast<int64_t>(F.size()) != N * B || G.size() != F.size())
            throw std::invalid_argument(adjoint ? "PCOp::apply_adjoint: shape mismatch" : "PCOp::apply: shape mismatch");
        check(adjoint ? pcb_apply_adjoint_batch(op_, B, F.data(), G.data()) : pcb_apply_batch(op_, B, F.data(), G.data()));
    }
    std::vector<double> apply_adjoint_batch(const std::vector<double>& F, int32_t B) const {
        return run(F, B, true);
    }

    // pc_operator.cpp:84-96
    double entry(const Point& y, const Point& x) const {
        double out = 0.0;
        check(pcb_entries(op_, 1, y.data(), x.data(), &out));
        return out;
    }

    // hmatrix.cpp:138-150 dense blocks, out[b][i][j]
    std::vector<double> blocks(const std::vector<int64_t>& t_origin, const std::vector<int64_t>& s_origin,
                               const Point& block_shape) const {
        const int32_t d = static_cast<int32_t>(domain_.lo.size());
        const int32_t nblk = static_cast<int32_t>(t_origin.size() / d);
        int64_t bs = 1;
        for (int64_t v : block_shape) bs *= v;
        std::vector<double> out(static_cast<size_t>(nblk) * bs * bs);
        check(pcb_blocks(op_, nblk, t_origin.data(), s_origin.data(), block_shape.data(), out.data()));
        return out;
    }

    pcb_op* handle() const { return op_; }

  private:
    std::vector<double> run(const std::vector<double>& F, int32_t B, bool adjoint) const {
        const int64_t N = domain_.num_points();
        if (static_cast<int64_t>(F.size()) != N * B)
            throw std::invalid_argument(adjoint ? "PCOp::apply_adjoint: shape mismatch"
                                                : "PCOp::apply: shape mismatch");
        std::vector<double> G(F.size());
        check(adjoint ? pcb_apply_adjoint_batch(op_, B, F.data(), G.data())
                      : pcb_apply_batch(op_, B, F.data(), G.data()));
        return G;
    }

    Box domain_;
    pcb_op* op_ = nullptr;
};

}  // namespace pcb

#endif  // PCB_OPERATOR_HPP
