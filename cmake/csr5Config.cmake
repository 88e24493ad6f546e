# csr5 CMake package over the B200 library (the reference's csr5::core,
# proj/core/CMakeLists.txt + cmake/csr5Config.cmake.in, README.md:110-123):
#
#   find_package(csr5 REQUIRED)            # -Dcsr5_DIR=<repo>/cmake
#   target_link_libraries(app PRIVATE csr5::core)
#
# csr5::core is libcsr5g.so (built in-tree by `make lib`, sm_100a) with the
# drop-in headers include/csr5/*.hpp (namespace csr5) and the C ABI
# include/csr5g.h.  C++20, as the reference.
get_filename_component(_csr5_root "${CMAKE_CURRENT_LIST_DIR}/.." ABSOLUTE)
set(_csr5_lib "${_csr5_root}/paper_1503_05032_b200/libcsr5g.so")
if(NOT EXISTS "${_csr5_lib}")
  set(csr5_FOUND FALSE)
  set(csr5_NOT_FOUND_MESSAGE "${_csr5_lib} is missing: run `make lib` in ${_csr5_root}")
  return()
endif()
if(NOT TARGET csr5::core)
  add_library(csr5::core SHARED IMPORTED)
  set_target_properties(csr5::core PROPERTIES
    IMPORTED_LOCATION "${_csr5_lib}"
    IMPORTED_SONAME "libcsr5g.so"
    INTERFACE_INCLUDE_DIRECTORIES "${_csr5_root}/include"
    INTERFACE_COMPILE_FEATURES cxx_std_20)
endif()
set(csr5_FOUND TRUE)
