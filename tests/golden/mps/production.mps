* a small bounded production plan with a range row and a free column;
* optimal, so the recovered solution is compared too
NAME          PROD
ROWS
 N  COST
 L  LAB
 L  MAT
 G  DEMA
 G  DEMB
 E  LINK
COLUMNS
    PA        COST      -5.0         LAB       2.0
    PA        MAT       1.0          DEMA      1.0
    PA        LINK      1.0
    PB        COST      -4.0         LAB       1.0
    PB        MAT       2.0          DEMB      1.0
    PC        COST      -3.5         LAB       1.5
    PC        MAT       1.5          DEMA      0.5
    PC        DEMB      0.5
    S         COST      0.25         LINK      -1.0
    T         COST      0.5          LINK      1.0
    T         MAT       -0.5
RHS
    RHS       LAB       100.0        MAT       80.0
    RHS       DEMA      5.0          DEMB      4.0
    RHS       LINK      2.0
RANGES
    RNG       LAB       60.0
BOUNDS
 UP BND       PA        30.0
 LO BND       PB        1.0
 UP BND       PC        25.0
 FR BND       T
 UP BND       S         10.0
ENDATA
