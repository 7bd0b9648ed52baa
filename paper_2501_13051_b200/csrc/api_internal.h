// Handle types behind the opaque pointers of include/fvlog.h and the
// exception -> status translation shared by the api_*.cpp translation units.
#pragma once

#include <memory>
#include <new>
#include <string>
#include <vector>

#include "column.h"
#include "fvlog.h"

namespace fv {
class Transport;
}

struct fv_ctx {
    fv::Ctx* c = nullptr;
    std::unique_ptr<fv::Transport> tx;  // partitioned evaluation (NCCL)
    ~fv_ctx();
};

struct fv_column {
    fv_ctx* ctx = nullptr;
    std::unique_ptr<fv::Column> owned;
    const fv::Column* col = nullptr;
};

struct fv_version {
    fv_ctx* ctx = nullptr;
    std::unique_ptr<fv::Version> v;
    std::vector<std::unique_ptr<fv_column>> views;
};

struct fv_relation {
    fv_ctx* ctx = nullptr;
    std::string name;
    uint32_t arity = 0;
    std::unique_ptr<fv_version> full, delta, new_rows;
};

struct fv_array {
    fv_ctx* ctx = nullptr;
    fv::Array a;
};

struct fv_match {
    fv_ctx* ctx = nullptr;
    std::unique_ptr<fv::Match> m;
};

namespace fvapi {

fv_status set_error(fv_ctx* ctx, fv_status s, const std::string& msg);
fv_version* wrap_version(fv_ctx* ctx, std::unique_ptr<fv::Version> v);
fv_array* wrap_array_u32(fv_ctx* ctx, fv::DBuf<fv::u32>&& b, fv::u64 n);

}  // namespace fvapi

#define FV_API_BEGIN(ctxp)               \
    fv_ctx* fv_api_ctx_ = (ctxp);        \
    try {                                \
        if (fv_api_ctx_) fv_api_ctx_->c->activate();

#define FV_API_END                                                                   \
    }                                                                                \
    catch (const fv::Error& e) {                                                     \
        return fvapi::set_error(fv_api_ctx_, e.status, e.what());                    \
    }                                                                                \
    catch (const std::bad_alloc&) {                                                  \
        return fvapi::set_error(fv_api_ctx_, FV_ERR_OOM, "host allocation failed");  \
    }                                                                                \
    catch (const std::exception& e) {                                                \
        return fvapi::set_error(fv_api_ctx_, FV_ERR_INVALID, e.what());              \
    }                                                                                \
    return FV_OK;

#define FV_REQUIRE(cond, status, msg) \
    do {                              \
        if (!(cond)) fv::fail(status, msg); \
    } while (0)
