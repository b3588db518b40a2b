// ORACLE TEST INFRASTRUCTURE — not product code.
//
// Restatement of the Eigen-light part of the reference operator seam
// (reference: proj/core/src/operators.cpp:13-49): OperatorHandle
// construction/apply/adjoint with atomic counters, to_grid_function and
// to_vector.  The rest of operators.cpp (example operators, Poisson-Schur
// with SimplicialLDLT) needs Eigen's sparse Cholesky and is not part of the
// apply path, so it is not built.  pou.cpp (harmonic weights, Eigen
// SimplicialLDLT) is replaced by a WeightBuilder that throws: the oracle
// only assembles operators from explicit weights/impulses (the reference
// constructor, pc_operator.cpp:26-38).
#include <algorithm>
#include <stdexcept>

#include "pcop/operators.hpp"
#include "pcop/pou.hpp"

namespace pcop {

OperatorHandle::OperatorHandle(IndexBox domain, ApplyFn apply, ApplyFn apply_adjoint,
                               EntryFn entry)
    : impl_(std::make_shared<Impl>()) {
    impl_->domain = std::move(domain);
    impl_->apply = std::move(apply);
    impl_->adjoint = std::move(apply_adjoint);
    impl_->entry = std::move(entry);
}

Eigen::VectorXd OperatorHandle::apply(const Eigen::VectorXd& f) const {
    if (f.size() != n()) throw std::invalid_argument("OperatorHandle::apply: size mismatch");
    impl_->n_apply.fetch_add(1);
    return impl_->apply(f);
}

Eigen::VectorXd OperatorHandle::apply_adjoint(const Eigen::VectorXd& f) const {
    if (f.size() != n())
        throw std::invalid_argument("OperatorHandle::apply_adjoint: size mismatch");
    impl_->n_adjoint.fetch_add(1);
    return impl_->adjoint(f);
}

void OperatorHandle::reset_counters() const {
    impl_->n_apply.store(0);
    impl_->n_adjoint.store(0);
}

GridFunction to_grid_function(const IndexBox& box, const Eigen::VectorXd& v) {
    if (v.size() != box.num_points()) throw std::invalid_argument("to_grid_function: size mismatch");
    GridFunction out(box);
    std::copy_n(v.data(), v.size(), out.data());
    return out;
}

Eigen::VectorXd to_vector(const GridFunction& f) {
    return Eigen::VectorXd(f.data(), static_cast<Eigen::Index>(f.size()));
}

// --- harmonic weights are out of the oracle's scope -----------------------
WeightBuilder::WeightBuilder(const AdaptiveGrid& grid, double tol) : grid_(&grid), tol_(tol) {}

WeightFunction WeightBuilder::build(int) {
    throw std::logic_error("oracle build: harmonic weights (pou.cpp) are not compiled");
}

void WeightBuilder::invalidate_cell(int cell_id) { cache_.erase(cell_id); }

}  // namespace pcop
