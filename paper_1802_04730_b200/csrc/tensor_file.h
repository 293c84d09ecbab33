// tensor_file.h — TCTN1 tensor files (tensor_file.cc).
#pragma once

#include <cstdint>
#include <string>
#include <vector>

#include "common.h"

namespace tcb {

struct TensorFile {
  bool isInt = false;
  std::vector<int64_t> shape;
  std::vector<uint32_t> bits;  // fp32 bit patterns or int32 values, row-major
};

void writeTensorFile(const std::string& path, const TensorFile& t);  // Error(Io)
TensorFile readTensorFile(const std::string& path);                  // Error(Io)

}  // namespace tcb
