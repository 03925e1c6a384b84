// Shared error reporting of libcurvigpu's translation units: records the
// thread-local message cg_last_error() returns and hands the code back.
#pragma once

int cg_internal_fail(int code, const char* msg);
