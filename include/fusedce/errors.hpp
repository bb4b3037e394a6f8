// Drop-in error taxonomy of the reference (proj/include/fusedce/errors.hpp:10-47):
// same enum order and exception names, so callers catch the same types.  The
// C-ABI reports fce_status = 1 + ErrorCode; throw_status() maps it back.
#pragma once

#include <stdexcept>
#include <string>

#include "fce/fce.h"

namespace fusedce {

enum class ErrorCode {
    DimensionMismatch,
    TargetOutOfRange,
    UnderflowRelease,
    DuplicateTarget,
    MissingStats,
    InconsistentUpstream,
    UnsupportedReduction,
    InvalidLayout,
    EmptyGrid,
    EmptyInput,
};

class Error : public std::runtime_error {
  public:
    Error(ErrorCode code, const std::string& what) : std::runtime_error(what), code_(code) {}
    ErrorCode code() const noexcept { return code_; }

  private:
    ErrorCode code_;
};

template <ErrorCode C>
class TypedError : public Error {
  public:
    explicit TypedError(const std::string& what) : Error(C, what) {}
};

using DimensionMismatch = TypedError<ErrorCode::DimensionMismatch>;
using TargetOutOfRange = TypedError<ErrorCode::TargetOutOfRange>;
using UnderflowRelease = TypedError<ErrorCode::UnderflowRelease>;
using DuplicateTarget = TypedError<ErrorCode::DuplicateTarget>;
using MissingStats = TypedError<ErrorCode::MissingStats>;
using InconsistentUpstream = TypedError<ErrorCode::InconsistentUpstream>;
using UnsupportedReduction = TypedError<ErrorCode::UnsupportedReduction>;
using InvalidLayout = TypedError<ErrorCode::InvalidLayout>;
using EmptyGrid = TypedError<ErrorCode::EmptyGrid>;
using EmptyInput = TypedError<ErrorCode::EmptyInput>;

// Device / runtime failures that have no reference counterpart.
class DeviceError : public std::runtime_error {
  public:
    using std::runtime_error::runtime_error;
};

inline void throw_status(fce_status s, const char* context = "") {
    if (s == FCE_OK) return;
    std::string msg = std::string(context) + (context[0] ? ": " : "") + fce_last_error();
    switch (s) {
        case FCE_DIMENSION_MISMATCH: throw DimensionMismatch(msg);
        case FCE_TARGET_OUT_OF_RANGE: throw TargetOutOfRange(msg);
        case FCE_UNDERFLOW_RELEASE: throw UnderflowRelease(msg);
        case FCE_DUPLICATE_TARGET: throw DuplicateTarget(msg);
        case FCE_MISSING_STATS: throw MissingStats(msg);
        case FCE_INCONSISTENT_UPSTREAM: throw InconsistentUpstream(msg);
        case FCE_UNSUPPORTED_REDUCTION: throw UnsupportedReduction(msg);
        case FCE_INVALID_LAYOUT: throw InvalidLayout(msg);
        case FCE_EMPTY_GRID: throw EmptyGrid(msg);
        case FCE_EMPTY_INPUT: throw EmptyInput(msg);
        default: throw DeviceError(std::string(fce_status_string(s)) + ": " + msg);
    }
}

}  // namespace fusedce
