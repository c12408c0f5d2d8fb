// Batched Jacobi-PCG over P2 windows (cg_p2.cu).
#pragma once

#include <vector>

#include "cg.cuh"

namespace mlg {

class CgBatchP2 {
 public:
  // systems: windows of L's dof grid (x0, y0, w, h, rhs); mask: strip systems
  // (dof in the system), else nullptr; bsrc: rhs-interleaved full vector.
  void setup(Ctx& c, const Level& L, std::vector<CgSys> systems, const unsigned char* mask,
             const double* bsrc, int bstride);
  CgResult solve(Ctx& c, double tol);
  const double* x() const { return X_.get(); }
  const CgSys* sys_dev() const { return sys_d_.get(); }
  const std::vector<CgSys>& systems() const { return sys_h_; }

 private:
  const Level* L_ = nullptr;
  const unsigned char* mask_ = nullptr;
  const double* bsrc_ = nullptr;
  int bstride_ = 1;
  long long rows_ = 0;
  int ntiles_ = 0;
  std::vector<CgSys> sys_h_;
  DevBuf<CgSys> sys_d_;
  DevBuf<int> tsys_, tt_, running_;
  DevBuf<double> X_, R_, P_, Q_, part_;
  DevBuf<unsigned char> ctl_;
};

}  // namespace mlg
