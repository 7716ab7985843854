// LinkSpec <-> the C-ABI's 31-double LinkSpec record (include/pardyn_c.h):
// [0] mass, [1..3] com, [4..12] inertia_rot row-major, [13..18] joint_screw
// (angular, linear), [19..27] home rotation row-major, [28..30] home
// translation -- the field order of LinkSpec (model.hpp:17-23) and of the
// JSON model files (model.hpp:72-77). Internal to libpardyn.so.
#pragma once

#include "../../include/pardyn/pardyn.hpp"
#include "../../include/pardyn_c.h"

namespace pardyn::detail {

// Smallest eigenvalue of a symmetric 3x3 (pardyn_model_io.cpp).
double sym3_min_eig(const Mat3& a);

inline void to_record(const LinkSpec& l, double* f) {
  f[0] = l.mass;
  for (int k = 0; k < 3; ++k) f[1 + k] = l.com(k);
  l.inertia_rot.toRowMajor(f + 4);
  for (int k = 0; k < 3; ++k) {
    f[13 + k] = l.joint_screw.angular(k);
    f[16 + k] = l.joint_screw.linear(k);
  }
  l.home_transform.rotation.toRowMajor(f + 19);
  for (int k = 0; k < 3; ++k) f[28 + k] = l.home_transform.translation(k);
}

inline LinkSpec from_record(const double* f) {
  LinkSpec l;
  l.mass = f[0];
  l.com = Vec3(f[1], f[2], f[3]);
  l.inertia_rot = Mat3::FromRowMajor(f + 4);
  l.joint_screw = Twist(Vec3(f[13], f[14], f[15]), Vec3(f[16], f[17], f[18]));
  l.home_transform.rotation = Mat3::FromRowMajor(f + 19);
  l.home_transform.translation = Vec3(f[28], f[29], f[30]);
  return l;
}

inline void append_records(const RobotChain& c, std::vector<double>& out) {
  const std::size_t at = out.size();
  out.resize(at + c.links.size() * PD_LINK_FIELDS);
  for (std::size_t i = 0; i < c.links.size(); ++i) to_record(c.links[i], out.data() + at + i * PD_LINK_FIELDS);
}

inline RobotChain chain_from_records(const double* rec, int n) {
  RobotChain c;
  c.links.reserve(static_cast<std::size_t>(n));
  for (int i = 0; i < n; ++i) c.links.push_back(from_record(rec + static_cast<std::size_t>(i) * PD_LINK_FIELDS));
  return c;
}

}  // namespace pardyn::detail
