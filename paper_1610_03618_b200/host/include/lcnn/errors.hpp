// Error taxonomy of the lcnn API (drop-in for the reference's errors.hpp).
// Every library failure derives from lcnn::Error; the C ABI's lcnn_status
// codes map one-to-one onto these classes (see throw_status in device.hpp).
#pragma once

#include <stdexcept>

namespace lcnn {

struct Error : std::runtime_error {
  using std::runtime_error::runtime_error;
};

#define LCNN_DECLARE_ERROR(Kind) \
  struct Kind : Error {          \
    using Error::Error;          \
  }

LCNN_DECLARE_ERROR(ShapeError);        // dims / windows / extents
LCNN_DECLARE_ERROR(IndexError);        // element access out of range
LCNN_DECLARE_ERROR(LayoutError);       // a kernel that does not exist for a layout
LCNN_DECLARE_ERROR(PlanError);         // transform / coarsening plan rules
LCNN_DECLARE_ERROR(FormatError);       // T4D1 file format
LCNN_DECLARE_ERROR(DomainError);       // non-finite softmax input
LCNN_DECLARE_ERROR(UnsupportedError);  // e.g. FFT with stride > 1
LCNN_DECLARE_ERROR(ValidationError);   // network configs
LCNN_DECLARE_ERROR(CalibrationError);  // threshold calibration

#undef LCNN_DECLARE_ERROR

}  // namespace lcnn
