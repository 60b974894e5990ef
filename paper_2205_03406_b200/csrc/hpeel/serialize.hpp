// .hrep files (proj/include/hpeel/hmatrix.hpp:150-156, proj/src/serialize.cpp).
#pragma once

#include <memory>
#include <string>

#include "matrix.hpp"

namespace hpeel {

class H1Rep;
/// save_rep (serialize.cpp:156-188) for the H1 format, from the device rep.
void save_rep(const std::string& path, const H1Rep& rep);
/// load_rep (serialize.cpp:190-250) for the H1 format, onto `device`; the rep
/// carries the embedded tree. Other format tags: std::invalid_argument.
std::shared_ptr<H1Rep> load_rep(const std::string& path, int device);
void save_dense_matrix(const std::string& path, const Matrix& m);
Matrix load_dense_matrix(const std::string& path);

}  // namespace hpeel
